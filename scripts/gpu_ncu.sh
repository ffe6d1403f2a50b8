set -e
CMD="python bench.py --streams 8192 --steps 3 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:blocked -s 3 -c 1 -o gpurun_out/prof_blocked_v7 $CMD > gpurun_out/ncu_full.log 2>&1
