set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_partition.py -x -q > gpurun_out/pytest_part.log 2>&1; tail -5 gpurun_out/pytest_part.log
timeout 600 python scripts/c5_run.py --scale 22 --parts 2 --batch 100000 --batches 2 > gpurun_out/c5_s22.log 2>&1; cat gpurun_out/c5_s22.log | tail -5
timeout 900 python scripts/c5_run.py --scale 24 --parts 2 --batch 1000000 --batches 2 > gpurun_out/c5_s24.log 2>&1; cat gpurun_out/c5_s24.log | tail -5
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
timeout 1800 python scripts/c5_run.py --scale 26 --parts 4 --batch 1000000 --batches 2 > gpurun_out/c5_s26.log 2>&1; cat gpurun_out/c5_s26.log | tail -8
