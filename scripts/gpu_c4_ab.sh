for L in scratch/old def scratch/old def; do
  if [ "$L" = def ]; then P=""; else P=$PWD/$L/librgb.so; fi
  RGB_LIB_PATH=$P timeout 300 python bench.py --config c4 --steps 5 --warmup 2 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$L', d['ms_per_step'], d.get('parity'))"
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c4 or grid or random or wide or scaling or partial or continuation" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_reference_pins.py tests/test_experiments.py -q -m gpu -x 2>&1 | tail -1
