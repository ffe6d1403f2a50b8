set -o pipefail
timeout 300 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/c3_plain.json 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:panel_kernel -c 1 -o gpurun_out/c3_panel python bench.py --config c3 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_c3p.log 2>&1; tail -2 gpurun_out/ncu_c3p.log; tail -c 300 gpurun_out/c3_plain.json
