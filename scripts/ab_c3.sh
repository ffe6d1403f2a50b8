timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for so in scratch/variants/librgb_*.so; do RGB_LIB_PATH=$PWD/$so timeout 600 python bench.py --config c3 --steps 5 --warmup 2 --no-e2e --no-cpu 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$so', 'value %.4g' % d['value'], 'kernel_ms %.3f' % d['roofline']['kernel_ms'], 'parity', d['parity']['x_relerr_max'], d['parity']['rank_match'])"; done
