set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pushpull.py -m gpu -x -q > gpurun_out/pytest_pp.log 2>&1; tail -2 gpurun_out/pytest_pp.log
K="'' pp=1"
timeout 400 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 4 --knobs pp=1 > gpurun_out/ab39_C2.log 2>&1
timeout 400 python scripts/sweep.py --graph road --side 1024 --batch 10000 --batches 2 --knobs pp=1 > gpurun_out/ab39_road.log 2>&1
timeout 400 python scripts/sweep.py --graph rmat --scale 20 --batch 10000 --batches 4 --knobs pp=1 > gpurun_out/ab39_C3.log 2>&1
