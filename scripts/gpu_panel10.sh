bash scripts/ab_lib.sh scripts/kbench_c3.py def scratch/smsp
timeout 900 ncu --set full --import-source on --clock-control none -k regex:panel_kernel -c 1 -o gpurun_out/c3_panel3 python bench.py --config c3 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_c3p3.log 2>&1; tail -1 gpurun_out/ncu_c3p3.log
