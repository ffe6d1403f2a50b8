set -o pipefail
timeout 300 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/c3_plain.json 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:blocked_wg_kernel -c 1 -o gpurun_out/c3_wg python bench.py --config c3 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_c3.log 2>&1; tail -2 gpurun_out/ncu_c3.log
