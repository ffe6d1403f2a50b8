set -e
CMD="python bench.py --streams 8192 --steps 3 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain_c5small.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:blocked_kernel -s 3 -c 1 -o gpurun_out/prof_c5_r2 $CMD > gpurun_out/ncu_full_c5.log 2>&1
tail -2 gpurun_out/ncu_full_c5.log
