set -x
mkdir -p gpurun_out
K="'' bfs_local_max=16 bfs_local=8 bfs_local=-1"
eval timeout 400 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 4 --knobs $K > gpurun_out/sw5_C2.log 2>&1
eval timeout 300 python scripts/sweep.py --graph rmat --scale 20 --batch 10000 --batches 3 --knobs $K > gpurun_out/sw5_C3.log 2>&1
eval timeout 300 python scripts/sweep.py --graph road --side 1024 --batch 10000 --batches 2 --knobs $K > gpurun_out/sw5_road.log 2>&1
eval timeout 300 python scripts/sweep.py --graph random --batch 1000 --batches 3 --knobs $K > gpurun_out/sw5_C1.log 2>&1
python scripts/sweep_table.py gpurun_out/sw5_*.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
