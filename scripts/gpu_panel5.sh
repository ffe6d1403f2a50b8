bash scripts/ab_lib.sh scripts/kbench_c3.py def scratch/rcp1
RGB_LIB_PATH=$PWD/scratch/rcp1/librgb.so timeout 120 python scripts/panel_mismatch.py 2>&1 | tail -2
