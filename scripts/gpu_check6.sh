set -x
mkdir -p gpurun_out
timeout 400 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 4 --knobs '' 'pp=1' > gpurun_out/sw8_C2.log 2>&1
timeout 300 python scripts/sweep.py --graph rmat --scale 20 --batch 10000 --batches 3 --knobs '' 'pp=1' > gpurun_out/sw8_C3.log 2>&1
timeout 300 python scripts/sweep.py --graph road --side 1024 --batch 10000 --batches 2 --knobs '' 'pp=1' > gpurun_out/sw8_road.log 2>&1
timeout 300 python scripts/sweep.py --graph random --batch 1000 --batches 3 --knobs '' 'pp=1' > gpurun_out/sw8_C1.log 2>&1
python scripts/sweep_table.py gpurun_out/sw8_*.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-700
