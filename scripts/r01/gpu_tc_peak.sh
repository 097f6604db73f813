export A4_SHAPES="8192,8192,2048;8192,8192,4096;8192,8192,8192;16384,16384,4096"
for v in 1 0; do
POS_SFB_PAIR=$v TAG=pair$v timeout 200 python scripts/a4_bench.py 2>&1 | grep '^{' | grep -v '"KP": 0'
done
