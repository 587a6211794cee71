set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for rep in 1 2; do
for lib in old new; do
  if [ $lib = old ]; then export MFX_LIB_PATH=$PWD/build/old/libmfx.so; else unset MFX_LIB_PATH; fi
  timeout 300 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 4 --knobs '' > gpurun_out/ab28_${lib}_${rep}_C2.log 2>&1
  timeout 300 python scripts/sweep.py --graph road --side 1024 --batch 10000 --batches 2 --knobs '' > gpurun_out/ab28_${lib}_${rep}_road.log 2>&1
  timeout 300 python scripts/sweep.py --graph rmat --scale 20 --batch 10000 --batches 4 --knobs '' > gpurun_out/ab28_${lib}_${rep}_C3.log 2>&1
  timeout 300 python scripts/sweep.py --graph random --batch 1000 --batches 6 --knobs '' MFX_BFS_LOCAL_MAX=16 MFX_BFS_LOCAL=8 > gpurun_out/ab28_${lib}_${rep}_C1.log 2>&1
done
done
MFX_TRACE_CAP=400000 timeout 300 python scripts/trace.py --side 2048 > gpurun_out/trace_C2.log 2>&1
