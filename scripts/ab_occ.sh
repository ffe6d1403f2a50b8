for i in 1 2; do
  python scripts/kbench.py 16384 | cut -c1-60,170-230 | sed 's/^/minb3 /'
  RGB_LIB_PATH=$PWD/scratch/v3/librgb.so python scripts/kbench.py 16384 | cut -c1-60,170-230 | sed 's/^/minb2 /'
  RGB_LIB_PATH=$PWD/scratch/v2/librgb.so python scripts/kbench.py 16384 | cut -c1-60,170-230 | sed 's/^/minb1 /'
done
