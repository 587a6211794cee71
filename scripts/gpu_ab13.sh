set -x
mkdir -p gpurun_out
K="MFX_BFS_LOCAL=128 MFX_BFS_LOCAL=256 MFX_BFS_LOCAL=512 MFX_BFS_LOCAL=4096 MFX_BFS_LOCAL=256,MFX_LQ_CAP=1024"
eval timeout 400 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 4 --knobs $K > gpurun_out/ab14_C2.log 2>&1
eval timeout 400 python scripts/sweep.py --graph road --side 1024 --batch 10000 --batches 2 --knobs $K > gpurun_out/ab14_road.log 2>&1
eval timeout 400 python scripts/sweep.py --graph rmat --scale 20 --batch 10000 --batches 4 --knobs $K > gpurun_out/ab14_C3.log 2>&1
eval timeout 400 python scripts/sweep.py --graph random --batch 1000 --batches 6 --knobs $K > gpurun_out/ab14_C1.log 2>&1
