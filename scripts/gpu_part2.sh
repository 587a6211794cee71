set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_partition.py -x -q > gpurun_out/pytest_part.log 2>&1; tail -3 gpurun_out/pytest_part.log
timeout 900 python scripts/c5_run.py --scale 26 --parts 4 --batch 1000000 --batches 2 > gpurun_out/c5_phases.log 2>&1; cat gpurun_out/c5_phases.log
