timeout 60 python scripts/panel_check.py 2>&1 | tail -6; echo "check rc $?"
timeout 60 python scripts/panel_mismatch.py 2>&1 | tail -2
bash scripts/ab_lib.sh scripts/kbench_c3.py scratch/old def
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c3 or variants or fp32_inputs or partial or nonfinite or rank_cap or continuation or deterministic or random or other_inst or panel" 2>&1 | tail -3
timeout 120 python scripts/probe_panel.py 2>&1 | grep -E "^ms|P |H |scan"
