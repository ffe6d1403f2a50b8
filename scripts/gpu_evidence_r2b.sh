# session evidence: tests, smoke, bench lines for every config, default launch list
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
for c in c1 c2 c3 c4; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
python bench.py --dtype fp32 > gpurun_out/bench_c5_fp32.json 2> gpurun_out/bench_c5_fp32.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
for f in default c1 c2 c3 c4 c5_fp32 reference; do python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_$f.json').read().strip().splitlines()[-1]); r=d.get('roofline') or {}
print('$f', d.get('value'), d.get('ms_per_step'), r.get('frac'), (d.get('e2e') or {}).get('value'), (d.get('clocks') or {}).get('sm_mhz'))"; done
