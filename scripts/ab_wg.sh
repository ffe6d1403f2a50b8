for i in 1 2; do
  (cd scratch/old_tree && python scripts/kbench_c3.py | cut -c1-40 | sed 's/^/old  /')
  python scripts/kbench_c3.py | cut -c1-40 | sed 's/^/def  /'
  RGB_LIB_PATH=$PWD/scratch/f2/librgb.so python scripts/kbench_c3.py | cut -c1-40 | sed 's/^/f2   /'
  RGB_LIB_PATH=$PWD/scratch/f3/librgb.so python scripts/kbench_c3.py | cut -c1-40 | sed 's/^/f3   /'
done
for L in f2 f3; do RGB_LIB_PATH=$PWD/scratch/$L/librgb.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c3 or c1 or variants or fp32_inputs or partial or nonfinite or rank_cap or continuation or deterministic or random" 2>&1 | tail -1 | sed "s/^/$L tests: /"; done
