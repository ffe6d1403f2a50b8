# round-2 evidence: the default bench line, the ncu launch list of the same command,
# and per-config bench lines (each after the plain command exited 0)
set -e
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_default.csv python bench.py > gpurun_out/ncu_launch_run.log 2>&1
for c in c1 c2 c3 c4; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
python bench.py --dtype fp32 > gpurun_out/bench_c5_fp32.json 2> gpurun_out/bench_c5_fp32.err
tail -c 600 gpurun_out/bench_default.json
