set -x
mkdir -p gpurun_out
timeout 300 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 4 --knobs '' 'bfs_local_max=256' > gpurun_out/sw10_C2.log 2>&1
timeout 300 python scripts/sweep.py --graph rmat --scale 20 --batch 10000 --batches 3 --knobs '' > gpurun_out/sw10_C3.log 2>&1
timeout 300 python scripts/sweep.py --graph road --side 1024 --batch 10000 --batches 2 --knobs '' 'bfs_local_max=256' > gpurun_out/sw10_road.log 2>&1
timeout 300 python scripts/sweep.py --graph random --batch 1000 --batches 3 --knobs '' > gpurun_out/sw10_C1.log 2>&1
python scripts/sweep_table.py gpurun_out/sw10_*.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
