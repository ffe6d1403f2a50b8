set -o pipefail
bash scripts/ab_old_new.sh 2>&1 | cut -c1-200
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
