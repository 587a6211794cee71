set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python scripts/sweep.py --graph random --batch 1000 --batches 6 --knobs '' > gpurun_out/c16_C1.log 2>&1
timeout 300 python scripts/sweep.py --graph rmat --scale 20 --batch 10000 --batches 4 --knobs '' pp=1 > gpurun_out/c16_C3.log 2>&1
timeout 300 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 4 --knobs '' > gpurun_out/c16_C2.log 2>&1
