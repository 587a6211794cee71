set -x
mkdir -p gpurun_out
K="'' kernel_cycles=2 kernel_cycles=10 kernel_cycles=20"
for rep in 1 2; do
eval timeout 400 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 6 --knobs $K > gpurun_out/ab37_${rep}_C2.log 2>&1
done
eval timeout 400 python scripts/sweep.py --graph road --side 1024 --batch 10000 --batches 2 --knobs $K > gpurun_out/ab37_1_road.log 2>&1
