O=gpurun_out/r02/nvml; mkdir -p $O
nvidia-smi nvlink -h > $O/nvlink_help.txt 2>&1
nvidia-smi nvlink -gt d -i 0 > $O/gt_before.txt 2>&1
python scripts/r02/nvml_probe.py > $O/probe.txt 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29941 scripts/nvlink_peaks.py $O/np.json > /dev/null 2>&1
nvidia-smi nvlink -gt d -i 0 > $O/gt_after.txt 2>&1
python scripts/r02/nvml_probe.py > $O/probe_after.txt 2>&1
head -30 $O/gt_before.txt; head -30 $O/gt_after.txt; cat $O/probe.txt $O/probe_after.txt; grep -i "throughput\|-gt\|counter" $O/nvlink_help.txt | head
