set -o pipefail
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for c in c1; do timeout 900 python bench.py --config $c --steps 5 --warmup 2 --no-e2e 2>&1 | tail -1 > gpurun_out/bench_$c.json; python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', 'value %.4g' % d['value'], 'ms/step %.3f' % d['ms_per_step'], 'frac', d['roofline']['frac'], 'cpu', d['cpu_baseline'] and d['cpu_baseline']['value'], 'parity', d['parity'], d['status'])"; done
