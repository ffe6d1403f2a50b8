set -o pipefail
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "grid_kernel" 2>&1 | tail -15
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
for c in c2 c4; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 > gpurun_out/bench_$c.json; python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', 'value %.4g' % d['value'], 'ms/step %.3f' % d['ms_per_step'], 'frac %.4f' % d['roofline']['frac'], 'parity', d['parity'])"; done
