# final-ish evidence: bench line, ncu launch list of the same command, one full capture of the C5 kernel
set -e
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_default.csv python bench.py > gpurun_out/ncu_launch_run.log 2>&1
CMD="python bench.py --streams 8192 --steps 3 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain_small.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:blocked_kernel -s 3 -c 1 -o gpurun_out/prof_blocked_r1b $CMD > gpurun_out/ncu_full.log 2>&1
CMD3="python bench.py --config c3 --steps 3 --warmup 2 --no-e2e --no-cpu"
$CMD3 > gpurun_out/plain_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:blocked_wg -s 2 -c 1 -o gpurun_out/prof_wg_r1 $CMD3 > gpurun_out/ncu_full_c3.log 2>&1
