timeout 300 python bench.py --config c4 --steps 1 --warmup 2 --no-e2e --no-cpu > gpurun_out/c4_plain.json 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:grid_kernel -c 1 -o gpurun_out/c4_grid python bench.py --config c4 --steps 1 --warmup 2 --no-e2e --no-cpu > gpurun_out/ncu_c4.log 2>&1; tail -1 gpurun_out/ncu_c4.log
