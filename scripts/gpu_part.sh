set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_partition.py -x -q > gpurun_out/pytest_part.log 2>&1; tail -30 gpurun_out/pytest_part.log
