set -x
mkdir -p gpurun_out
K="'' MFX_TAIL_TIME=16 MFX_TAIL_TIME=24 MFX_TAIL_TIME=40 MFX_TAIL_TIME=80"
for rep in 1 2; do
eval timeout 400 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 6 --knobs $K > gpurun_out/ab19_${rep}_C2.log 2>&1
done
eval timeout 400 python scripts/sweep.py --graph road --side 1024 --batch 10000 --batches 2 --knobs $K > gpurun_out/ab19_1_road.log 2>&1
MFX_TAIL_TIME=24 MFX_TRACE_CAP=400000 timeout 300 python scripts/trace.py --side 2048 > gpurun_out/trace_C2.log 2>&1
