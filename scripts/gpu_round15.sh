set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "cluster or grid or capacity or dropin" > gpurun_out/t15.log 2>&1; echo "tests rc=$?" >> gpurun_out/t15.log
python bench.py --config c2 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/b15_c2.log 2>&1
python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/b15_c4.log 2>&1
python scripts/scaling_experiments.py gpurun_out > gpurun_out/scaling15.log 2>&1
