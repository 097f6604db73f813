# A/B at P=2: round-1 library+bench vs current (trace / no-trace / NVLS CTA variants)
mkdir -p gpurun_out/r02/ab
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
run() { name=$1; shift; timeout 300 "$@" > gpurun_out/r02/ab/$name.json 2> gpurun_out/r02/ab/$name.err; echo "$name rc=$? $(python -c "import json,sys; d=json.loads(open('gpurun_out/r02/ab/$name.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['roofline']['kernel_ms_per_step'],4))" 2>/dev/null)"; }
run r1 bash -c "cd build/r1_tree && $T --master-port 29601 bench.py --gpus 2 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e"
run cur $T --master-port 29602 bench.py --gpus 2 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-tf32
run cur_notrace $T --master-port 29603 bench.py --gpus 2 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-tf32 --no-trace
POS_NVLS_CTAS=32 run cur_c32 $T --master-port 29604 bench.py --gpus 2 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-tf32
POS_NVLS_CTAS=128 run cur_c128 $T --master-port 29605 bench.py --gpus 2 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-tf32
run r1_layers bash -c "cd build/r1_tree && $T --master-port 29606 bench.py --gpus 2 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --layers"
grep -v "^\[" gpurun_out/r02/ab/r1_layers.err | tail -9
