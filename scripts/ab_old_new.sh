# same-box A/B: HEAD build in scratch/old_tree vs the working tree (C5 blocked kernel, C3 warp-group kernel)
for i in 1 2; do
  (cd scratch/old_tree && python scripts/kbench.py 16384 | tail -1 | cut -c1-220 | sed 's/^/old /')
  python scripts/kbench.py 16384 | tail -1 | cut -c1-220 | sed 's/^/new /'
  (cd scratch/old_tree && python scripts/kbench_c3.py | tail -1 | sed 's/^/old /')
  python scripts/kbench_c3.py | tail -1 | sed 's/^/new /'
done
