set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_partition.py -x -q > gpurun_out/pytest_part.log 2>&1; tail -3 gpurun_out/pytest_part.log
for d in 0 4 16 64; do
  MFX_PART_BOTTOM_UP=$d timeout 900 python scripts/c5_run.py --scale 24 --parts 2 --batch 1000000 --batches 2 > gpurun_out/bu_s24_$d.log 2>&1
done
for d in 0 16; do
  MFX_PART_BOTTOM_UP=$d timeout 1800 python scripts/c5_run.py --scale 26 --parts 4 --batch 1000000 --batches 2 > gpurun_out/bu_s26_$d.log 2>&1
done
