timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 120 python scripts/probe_panel.py 2>&1 | grep -E "^ms|row mode|projection|wait|scan"
timeout 300 python bench.py --config c3 --steps 10 --warmup 3 > gpurun_out/bench_c3_panel3.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/bench_c3_panel3.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'])"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
