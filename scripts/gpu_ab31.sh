set -x
mkdir -p gpurun_out
K="'' MFX_BFS_LOCAL_MAX=256 MFX_BFS_LOCAL_MAX=100000 pp=1 pp=1,MFX_BFS_LOCAL_MAX=256 pp=1,MFX_BFS_LOCAL_MAX=100000"
eval timeout 400 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 4 --knobs $K > gpurun_out/ab31_C2.log 2>&1
eval timeout 400 python scripts/sweep.py --graph rmat --scale 20 --batch 10000 --batches 4 --knobs $K > gpurun_out/ab31_C3.log 2>&1
eval timeout 400 python scripts/sweep.py --graph random --batch 1000 --batches 4 --knobs $K > gpurun_out/ab31_C1.log 2>&1
eval timeout 400 python scripts/sweep.py --graph road --side 1024 --batch 10000 --batches 2 --knobs $K > gpurun_out/ab31_road.log 2>&1
