timeout 120 python scripts/probe_panel.py 2>&1 | tail -24
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dl tools/dmma_latency.cu && for c in 1 2 4 8; do /tmp/dl $c 1; done 2>&1 | tail -8
