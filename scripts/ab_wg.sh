for i in 1 2; do
  (cd scratch/old_tree && python scripts/kbench_c3.py | sed 's/^/old /')
  python scripts/kbench_c3.py | sed 's/^/new /'
done
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c3 or c1 or variants or fp32_inputs or partial or nonfinite or rank_cap or continuation or deterministic" 2>&1 | tail -2
