set -o pipefail
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "fp32_inputs" 2>&1 | tail -15
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 600 python bench.py --no-e2e --no-cpu 2>&1 | tail -1 > gpurun_out/bench_c5.json; python -c "
import json; d=json.load(open('gpurun_out/bench_c5.json')); print('c5 value %.4g' % d['value'], 'ms/step %.3f' % d['ms_per_step'], 'frac %.4f' % d['roofline']['frac'], 'parity', d['parity'])"
