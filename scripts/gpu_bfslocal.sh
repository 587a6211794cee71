set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
K="bfs_local=-1 bfs_local=2 bfs_local=4 bfs_local=8 bfs_local=16 bfs_local=32"
timeout 300 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 3 --knobs $K > gpurun_out/bl_C2.log 2>&1
timeout 300 python scripts/sweep.py --graph rmat --scale 20 --batch 10000 --batches 3 --knobs $K > gpurun_out/bl_C3.log 2>&1
timeout 300 python scripts/sweep.py --graph random --batch 1000 --batches 3 --knobs $K > gpurun_out/bl_C1.log 2>&1
MFX_TIMEOUT_S=120 timeout 600 python scripts/sweep.py --graph road --side 1024 --batch 10000 --batches 2 --knobs $K 'bfs_local=64' 'bfs_local=32,schedule=async' > gpurun_out/bl_road1024.log 2>&1
cat gpurun_out/bl_*.log | cut -c1-400
