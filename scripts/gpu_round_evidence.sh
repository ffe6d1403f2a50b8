# round evidence: the default bench line, the ncu launch list of the same command,
# per-config bench lines, and one ncu capture per tensor-core kernel (each after
# its plain command exited 0)
set -e
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_default.csv python bench.py > gpurun_out/ncu_launch_run.log 2>&1
for c in c1 c2 c3 c4; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
python bench.py --dtype fp32 > gpurun_out/bench_c5_fp32.json 2> gpurun_out/bench_c5_fp32.err
CMD="python bench.py --streams 8192 --steps 3 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain_c5small.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:blocked_kernel -s 3 -c 1 -o gpurun_out/prof_c5_r2 $CMD > gpurun_out/ncu_c5.log 2>&1
CMD2="python bench.py --config c2 --steps 1 --warmup 3 --no-e2e --no-cpu"
$CMD2 > gpurun_out/plain_c2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:cluster_kernel -s 3 -c 1 -o gpurun_out/prof_c2_r2 $CMD2 > gpurun_out/ncu_c2.log 2>&1
tail -c 400 gpurun_out/bench_default.json
