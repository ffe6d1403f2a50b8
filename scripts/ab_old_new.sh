# same-box A/B of the C5 blocked kernel: HEAD build in scratch/old_tree vs the working tree
for i in 1 2; do
  (cd scratch/old_tree && python scripts/kbench.py 16384 | tail -1 | sed 's/^/old /')
  python scripts/kbench.py 16384 | tail -1 | sed 's/^/new /'
done
