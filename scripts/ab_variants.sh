# A/B the kernel variants under scratch/variants (same bench command, kernel ms)
for so in scratch/variants/librgb_*.so; do
  name=$(basename $so .so)
  RGB_LIB_PATH=$PWD/$so python bench.py --streams 32768 --steps 3 --warmup 2 --no-e2e --no-cpu 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$name', 'rows/s %.3e' % d['value'], 'kernel_ms %.3f' % r['kernel_ms'], 'frac %.3f' % r['frac'], 'parity', d['parity']['x_relerr_max'])"
done
