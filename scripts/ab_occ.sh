for i in 1 2; do
  python scripts/kbench.py 16384 | cut -c1-40,170-230 | sed 's/^/w4 /'
  RGB_LIB_PATH=$PWD/scratch/v2/librgb.so python scripts/kbench.py 16384 | cut -c1-40,170-230 | sed 's/^/w2 /'
  RGB_LIB_PATH=$PWD/scratch/v3/librgb.so python scripts/kbench.py 16384 | cut -c1-40,170-230 | sed 's/^/w6 /'
done
