for so in scratch/variants/librgb_*.so; do RGB_LIB_PATH=$PWD/$so python scripts/kbench.py 16384; RGB_LIB_PATH=$PWD/$so python scripts/kbench.py 16384; done
