set -x
mkdir -p gpurun_out
K="'' device_flags=4 MFX_WAVE_TIME=6 MFX_WAVE_TIME=14"
for rep in 1 2; do
eval timeout 400 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 6 --knobs $K > gpurun_out/ab34_${rep}_C2.log 2>&1
done
