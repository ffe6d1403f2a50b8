set -o pipefail
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "cluster or grid_kernel or c2" 2>&1 | tail -2
for i in 1 2; do timeout 600 python bench.py --config c2 --steps 10 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 > gpurun_out/bench_c2.json; python -c "
import json; d=json.load(open('gpurun_out/bench_c2.json')); print('c2 value %.4g' % d['value'], 'ms/step %.3f' % d['ms_per_step'], 'parity', d['parity'])"; done
