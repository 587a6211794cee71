set -x
mkdir -p gpurun_out
K="'' MFX_RING_SLEEP=0 MFX_RING_SLEEP=16 MFX_RING_SLEEP=256 MFX_RING_SLEEP=1000"
for rep in 1 2; do
eval timeout 400 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 6 --knobs $K > gpurun_out/ab36_${rep}_C2.log 2>&1
done
eval timeout 400 python scripts/sweep.py --graph road --side 1024 --batch 10000 --batches 2 --knobs $K > gpurun_out/ab36_1_road.log 2>&1
