timeout 300 python bench.py --config c3 --steps 10 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_c3.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks'])"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:panel_kernel -c 1 -o gpurun_out/c3_panel4 python bench.py --config c3 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_c3p4.log 2>&1; tail -1 gpurun_out/ncu_c3p4.log
