# first try of the panel kernel: quick parity probe, C3 timing A/B vs the warp-group kernel, parity tests
timeout 120 python scripts/panel_check.py > gpurun_out/panel_check.log 2>&1; echo "check exit $?" >> gpurun_out/panel_check.log
cat gpurun_out/panel_check.log | tail -20
for i in 1 2; do
  RGB_NO_PANEL=1 timeout 120 python scripts/kbench_c3.py | cut -c1-60 | sed 's/^/wg    /'
  timeout 120 python scripts/kbench_c3.py | cut -c1-60 | sed 's/^/panel /'
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c3 or variants or fp32_inputs or partial or nonfinite or rank_cap or continuation or deterministic or random" 2>&1 | tail -15
