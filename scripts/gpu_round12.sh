set -o pipefail
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "cluster or grid_kernel or c2 or fp32_inputs" 2>&1 | tail -5
timeout 600 ncu --set full --import-source on -k regex:cluster_kernel -c 1 -o gpurun_out/c2_cluster python bench.py --config c2 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_c2.log 2>&1; tail -3 gpurun_out/ncu_c2.log
