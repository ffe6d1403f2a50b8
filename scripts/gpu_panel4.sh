timeout 120 python scripts/panel_mismatch.py 2>&1 | tail -2
timeout 120 python scripts/probe_panel.py 2>&1 | tail -22
RGB_NO_PANEL=1 timeout 120 python scripts/kbench_c3.py | cut -c1-50 | sed 's/^/wg     /'
bash scripts/ab_lib.sh scripts/kbench_c3.py def scratch/smsp scratch/stdldl
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c3 or variants or fp32_inputs or partial or nonfinite or rank_cap or continuation or deterministic or random" 2>&1 | tail -3
