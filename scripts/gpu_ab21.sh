set -x
mkdir -p gpurun_out
K="'' device_flags=1 device_flags=2"
for rep in 1 2; do
eval timeout 400 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 6 --knobs $K > gpurun_out/ab21_${rep}_C2.log 2>&1
done
eval timeout 400 python scripts/sweep.py --graph road --side 1024 --batch 10000 --batches 2 --knobs $K > gpurun_out/ab21_1_road.log 2>&1
eval timeout 400 python scripts/sweep.py --graph rmat --scale 20 --batch 10000 --batches 4 --knobs $K > gpurun_out/ab21_1_C3.log 2>&1
