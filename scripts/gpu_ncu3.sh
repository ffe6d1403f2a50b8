set -e
CMD="python bench.py --config c3 --steps 3 --warmup 2 --no-e2e --no-cpu"
$CMD > gpurun_out/plain_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:blocked_wg -s 2 -c 1 -o gpurun_out/prof_wg_v1 $CMD > gpurun_out/ncu_full_c3.log 2>&1
