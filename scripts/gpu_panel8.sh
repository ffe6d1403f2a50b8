bash scripts/ab_lib.sh scripts/kbench_c3.py def scratch/cta3
RGB_LIB_PATH=$PWD/scratch/cta3/librgb.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c3 or variants or fp32_inputs or partial or nonfinite or rank_cap or continuation or deterministic or random or other_inst" 2>&1 | tail -2
