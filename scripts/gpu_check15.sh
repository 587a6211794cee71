set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for rep in 1 2; do
timeout 300 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 4 --knobs '' > gpurun_out/c15_${rep}_C2.log 2>&1
timeout 300 python scripts/sweep.py --graph road --side 1024 --batch 10000 --batches 2 --knobs '' > gpurun_out/c15_${rep}_road.log 2>&1
done
timeout 300 python scripts/sweep.py --graph rmat --scale 20 --batch 10000 --batches 3 --knobs '' pp=1 > gpurun_out/c15_1_C3.log 2>&1
MFX_TRACE_CAP=400000 timeout 300 python scripts/trace.py --side 2048 > gpurun_out/trace_C2.log 2>&1
