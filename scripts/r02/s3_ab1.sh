# P=1 A/B: round-1 tree vs current (with / without device tracing), alternating, 3 rounds; then the A4 profile set
mkdir -p gpurun_out/r02/ab1
run() { name=$1; shift; timeout 300 "$@" > gpurun_out/r02/ab1/$name.json 2> gpurun_out/r02/ab1/$name.err; echo "$name rc=$? $(python -c "import json,sys; d=json.loads(open('gpurun_out/r02/ab1/$name.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['roofline']['kernel_ms_per_step'],4), d['clocks'])" 2>/dev/null)"; }
for i in 1 2 3; do
run r1_$i bash -c "cd build/r1_tree && python bench.py --steps 50 --warmup 10 --no-cpu-baseline --no-e2e"
run cur_$i python bench.py --steps 50 --warmup 10 --no-cpu-baseline --no-e2e --no-tf32
run curnt_$i python bench.py --steps 50 --warmup 10 --no-cpu-baseline --no-e2e --no-tf32 --no-trace
done
bash scripts/r02/s3_a4prof.sh
