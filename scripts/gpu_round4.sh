set -o pipefail
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for c in c2 c4; do timeout 900 python bench.py --config $c --steps 5 --warmup 2 --no-e2e 2>&1 | tail -1 > gpurun_out/bench_$c.json; python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', 'value %.4g' % d['value'], 'ms/step %.3f' % d['ms_per_step'], 'frac %.4f' % d['roofline']['frac'], 'cpu', d['cpu_baseline'] and d['cpu_baseline']['value'], d['cpu_baseline']['sample'], 'parity', d['parity'], d['config']['l2'])"; done
