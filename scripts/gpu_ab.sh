set -o pipefail
bash scripts/ab_old_new.sh 2>&1 | cut -c1-250
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c5 or golden or kahan or known" 2>&1 | tail -2
