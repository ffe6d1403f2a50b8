set -e
for spec in "c4 grid_kernel 1" "c3 blocked_wg_kernel 3" "c1 blocked_wg_kernel 3"; do
  set -- $spec
  CMD="python bench.py --config $1 --steps 1 --warmup 3 --no-e2e --no-cpu"
  $CMD > gpurun_out/plain_$1.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -o gpurun_out/prof_$1_r2 $CMD > gpurun_out/ncu_$1.log 2>&1
  tail -1 gpurun_out/ncu_$1.log
done
