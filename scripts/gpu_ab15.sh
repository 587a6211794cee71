set -x
mkdir -p gpurun_out
K="'' MFX_SCHEDULE=async MFX_SCHEDULE=async,async_budget=4 MFX_SCHEDULE=async,async_budget=64 MFX_TAIL_LOCAL=1024 MFX_TAIL_LOCAL=4096"
eval timeout 400 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 4 --knobs $K > gpurun_out/ab15_C2.log 2>&1
eval timeout 400 python scripts/sweep.py --graph road --side 1024 --batch 10000 --batches 2 --knobs $K > gpurun_out/ab15_road.log 2>&1
eval timeout 400 python scripts/sweep.py --graph rmat --scale 20 --batch 10000 --batches 4 --knobs $K > gpurun_out/ab15_C3.log 2>&1
