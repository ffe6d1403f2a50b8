timeout 120 python scripts/panel_mismatch.py 2>&1 | tail -3
timeout 120 python scripts/probe_panel.py 2>&1 | tail -24
for i in 1 2; do timeout 120 python scripts/kbench_c3.py | cut -c1-60 | sed 's/^/panel /'; done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c3 or variants or fp32_inputs or partial or nonfinite or rank_cap or continuation or deterministic or random" 2>&1 | tail -4
