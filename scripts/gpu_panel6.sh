timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python bench.py --config c3 --steps 10 --warmup 3 > gpurun_out/bench_c3_panel.json 2> gpurun_out/bench_c3_panel.err; tail -c 700 gpurun_out/bench_c3_panel.json
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
