set -x
mkdir -p gpurun_out
K="'' MFX_WAVE_TIME=4 MFX_WAVE_TIME=8 MFX_WAVE_TIME=12 MFX_WAVE_TIME=16 MFX_WAVE_TIME=8,wave_mult=4,wave_add=16"
eval timeout 400 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 4 --knobs $K > gpurun_out/ab17_C2.log 2>&1
eval timeout 400 python scripts/sweep.py --graph road --side 1024 --batch 10000 --batches 2 --knobs $K > gpurun_out/ab17_road.log 2>&1
eval timeout 400 python scripts/sweep.py --graph rmat --scale 20 --batch 10000 --batches 4 --knobs $K > gpurun_out/ab17_C3.log 2>&1
eval timeout 400 python scripts/sweep.py --graph random --batch 1000 --batches 6 --knobs $K > gpurun_out/ab17_C1.log 2>&1
