for L in def scratch/c2nohome; do
  if [ "$L" = def ]; then P=""; else P=$PWD/$L/librgb.so; fi
  RGB_LIB_PATH=$P timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$L', d['ms_per_step'])"
done
