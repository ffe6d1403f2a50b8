for L in scratch/old def scratch/old def; do
  if [ "$L" = def ]; then P=""; else P=$PWD/$L/librgb.so; fi
  RGB_LIB_PATH=$P timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$L', d['ms_per_step'], d.get('parity'))"
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c2 or cluster or random or partial or continuation or variants" 2>&1 | tail -2
