set -x
mkdir -p gpurun_out
MFX_BFS_SPLIT=6 timeout 600 python -m pytest tests -m gpu -x -q -k "parity or large" > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
K="'' MFX_BFS_SPLIT=4 MFX_BFS_SPLIT=6 MFX_BFS_SPLIT=7"
for rep in 1 2; do
eval timeout 400 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 6 --knobs $K > gpurun_out/ab25_${rep}_C2.log 2>&1
done
eval timeout 400 python scripts/sweep.py --graph road --side 1024 --batch 10000 --batches 2 --knobs $K > gpurun_out/ab25_1_road.log 2>&1
eval timeout 400 python scripts/sweep.py --graph rmat --scale 20 --batch 10000 --batches 4 --knobs $K > gpurun_out/ab25_1_C3.log 2>&1
