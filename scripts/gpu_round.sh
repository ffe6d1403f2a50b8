# one GPU call: tests, smoke, a bench line (inputs/logs land in gpurun_out/)
set -o pipefail
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -4
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -25
timeout 900 python bench.py --steps 3 --warmup 3 2>&1 | tail -3 | tee gpurun_out/bench_c5.jsonl
