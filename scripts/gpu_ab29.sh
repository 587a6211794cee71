set -x
mkdir -p gpurun_out
K="'' device_flags=16"
for rep in 1 2; do
eval timeout 400 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 6 --knobs $K > gpurun_out/ab29_${rep}_C2.log 2>&1
eval timeout 400 python scripts/sweep.py --graph road --side 1024 --batch 10000 --batches 2 --knobs $K > gpurun_out/ab29_${rep}_road.log 2>&1
done
eval timeout 400 python scripts/sweep.py --graph rmat --scale 20 --batch 10000 --batches 4 --knobs $K > gpurun_out/ab29_1_C3.log 2>&1
eval timeout 400 python scripts/sweep.py --graph random --batch 1000 --batches 6 --knobs $K > gpurun_out/ab29_1_C1.log 2>&1
MFX_TRACE_CAP=400000 timeout 300 python scripts/trace.py --side 2048 > gpurun_out/trace_C2.log 2>&1
