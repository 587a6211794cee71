set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
K="'' MFX_WALK_DEPTH=1 MFX_WALK_DEPTH=1,MFX_WALK_MAX=512 MFX_WALK_DEPTH=1,MFX_WALK_MAX=128"
for rep in 1 2; do
  eval timeout 400 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 4 --knobs $K > gpurun_out/ab9_${rep}_C2.log 2>&1
  eval timeout 400 python scripts/sweep.py --graph rmat --scale 18 --batch 10000 --batches 4 --knobs $K > gpurun_out/ab9_${rep}_rmat.log 2>&1
done
timeout 400 python scripts/sweep.py --graph road --side 1024 --batch 10000 --batches 2 --knobs '' > gpurun_out/ab9_1_road.log 2>&1
MFX_WALK_DEPTH=1 MFX_WALK_MAX=128 MFX_TRACE_CAP=400000 timeout 300 python scripts/trace.py --side 2048 > gpurun_out/trace_C2w.log 2>&1
