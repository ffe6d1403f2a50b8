timeout 300 python bench.py --config c2 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/c2_plain.json 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:cluster_kernel -c 1 -o gpurun_out/c2_cluster python bench.py --config c2 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_c2.log 2>&1; tail -1 gpurun_out/ncu_c2.log
