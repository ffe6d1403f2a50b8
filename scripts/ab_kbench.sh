timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for so in scratch/variants/librgb_*.so; do RGB_LIB_PATH=$PWD/$so python scripts/kbench.py 16384; RGB_LIB_PATH=$PWD/$so python scripts/kbench.py 16384; done
