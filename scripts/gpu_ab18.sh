set -x
mkdir -p gpurun_out
K="'' MFX_WAVE_TIME=8 MFX_WAVE_TIME=10 MFX_WAVE_TIME=12"
for rep in 1 2; do
eval timeout 400 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 6 --knobs $K > gpurun_out/ab18_${rep}_C2.log 2>&1
eval timeout 400 python scripts/sweep.py --graph road --side 1024 --batch 10000 --batches 2 --knobs $K > gpurun_out/ab18_${rep}_road.log 2>&1
eval timeout 400 python scripts/sweep.py --graph rmat --scale 20 --batch 10000 --batches 4 --knobs $K > gpurun_out/ab18_${rep}_C3.log 2>&1
done
