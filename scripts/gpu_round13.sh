set -o pipefail
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c3 or variants or fp32_inputs or partial or nonfinite or rank_capacity" 2>&1 | tail -2
for i in 1 2; do timeout 600 python bench.py --config c3 --no-e2e --no-cpu 2>&1 | tail -1 > gpurun_out/bench_c3.json; python -c "
import json; d=json.load(open('gpurun_out/bench_c3.json')); print('c3 value %.4g' % d['value'], 'ms/step %.3f' % d['ms_per_step'], 'frac %.4f' % d['roofline']['frac'], 'parity', d['parity'])"; done
