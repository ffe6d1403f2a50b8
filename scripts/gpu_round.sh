set -x
free -g | head -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 600 python bench.py --streams 8192 --steps 2 --warmup 1 --no-cpu 2>&1 | tail -3
