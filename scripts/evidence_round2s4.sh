# Evidence run of build round 2, fourth session (one gpurun call): GPU tests, every bench line,
# forced-sequential comparisons, launch lists, ncu captures of the two batched kernels, parity sweep, smoke.
# Output under gpurun_out/s4h; tools/ncu_summary.py turns the captures into profiles/round2s4_*.
O=gpurun_out/s4h; mkdir -p $O
(time python -m pytest tests -m gpu -x -q --timeout 300) > $O/gputests.log 2>&1
python bench.py > $O/bench_c5.json 2> $O/bench_c5.err
python bench.py --dtype fp32 --no-cpu > $O/bench_c5_fp32in.json 2> $O/bench_c5_fp32in.err
for c in c1 c2 c3 c4; do python bench.py --config $c --no-cpu > $O/bench_$c.json 2> $O/bench_$c.err; done
RGB_BLOCKED_SEQ=1 python bench.py --no-cpu --no-e2e > $O/bench_c5_sequential.json 2> /dev/null
RGB_PANEL_SEQ=1 python bench.py --config c3 --no-cpu --no-e2e > $O/bench_c3_sequential.json 2> /dev/null
python bench.py --gpus 2 --dist-backend gloo --streams 8192 --no-cpu --no-e2e --steps 5 > $O/bench_c5_2ranks_1gpu.json 2> $O/bench_c5_2ranks.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_default.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > $O/ncu_launches.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_c3.csv python bench.py --config c3 --steps 2 --warmup 3 --no-cpu --no-e2e > $O/ncu_launches_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:blocked_kernel -s 2 -c 1 -o $O/c5_blocked python bench.py --streams 8192 --no-cpu --no-e2e --steps 1 --warmup 1 > $O/ncu_c5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:panel_kernel -s 2 -c 1 -o $O/c3_panel python bench.py --config c3 --no-cpu --no-e2e --steps 1 --warmup 1 > $O/ncu_c3.log 2>&1
python scripts/parity_sweep.py $O/parity_sweep.json > $O/parity_sweep.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
tail -3 $O/gputests.log; tail -3 $O/smoke.log
