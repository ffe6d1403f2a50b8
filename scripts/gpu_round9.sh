set -o pipefail
bash scripts/ab_old_new.sh 2>&1 | cut -c1-300
timeout 900 python bench.py --dtype fp32 --no-e2e > gpurun_out/bench_c5_fp32.json 2> gpurun_out/bench_c5_fp32.err; python -c "
import json; d=json.load(open('gpurun_out/bench_c5_fp32.json')); print(d['value'], d['cpu_baseline'])"
