set -x
mkdir -p gpurun_out
K="'' MFX_MAX_CTAS=148 MFX_MAX_CTAS=222"
for rep in 1 2; do
eval timeout 400 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 6 --knobs $K > gpurun_out/ab30_${rep}_C2.log 2>&1
done
eval timeout 400 python scripts/sweep.py --graph road --side 1024 --batch 10000 --batches 2 --knobs $K > gpurun_out/ab30_1_road.log 2>&1
