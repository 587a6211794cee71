mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_partition.py -m gpu -x -q > gpurun_out/pytest_part.log 2>&1; tail -3 gpurun_out/pytest_part.log
