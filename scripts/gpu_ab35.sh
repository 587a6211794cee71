set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for rep in 1 2; do
for lib in old new; do
  if [ $lib = old ]; then export MFX_LIB_PATH=$PWD/build/old/libmfx.so; else unset MFX_LIB_PATH; fi
  timeout 300 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 6 --knobs '' > gpurun_out/ab35_${lib}_${rep}_C2.log 2>&1
done
done
