set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_partition.py tests/test_partition_host.py -x -q > gpurun_out/pytest_part.log 2>&1; tail -3 gpurun_out/pytest_part.log
timeout 1800 python scripts/c5_run.py --scale 26 --parts 4 --batch 1000000 --batches 2 > gpurun_out/c5_s26.log 2>&1; cat gpurun_out/c5_s26.log | tail -8
