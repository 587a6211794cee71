set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pushpull.py -x -q > gpurun_out/pytest_pp.log 2>&1; tail -15 gpurun_out/pytest_pp.log
timeout 400 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 4 --knobs '' 'pp=1' > gpurun_out/sw7_C2.log 2>&1
timeout 300 python scripts/sweep.py --graph rmat --scale 20 --batch 10000 --batches 3 --knobs '' 'pp=1' > gpurun_out/sw7_C3.log 2>&1
timeout 300 python scripts/sweep.py --graph road --side 1024 --batch 10000 --batches 2 --knobs '' 'pp=1' > gpurun_out/sw7_road.log 2>&1
timeout 300 python scripts/sweep.py --graph random --batch 1000 --batches 3 --knobs '' 'pp=1' > gpurun_out/sw7_C1.log 2>&1
python scripts/sweep_table.py gpurun_out/sw7_*.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
