set -e
CMD="python bench.py --streams 8192 --steps 2 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:blocked -s 1 -c 1 -o gpurun_out/prof_blocked_v5 $CMD > gpurun_out/ncu_full.log 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu 2>&1 | tail -1 > gpurun_out/bench_v5.json
