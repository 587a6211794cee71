set -x
mkdir -p gpurun_out
K="'' MFX_WAVE_TIME=8 MFX_WAVE_TIME=12 MFX_WAVE_TIME=16"
for rep in 1 2; do
eval timeout 400 python scripts/sweep.py --graph random --batch 1000 --batches 6 --knobs $K > gpurun_out/ab38_${rep}_C1.log 2>&1
done
