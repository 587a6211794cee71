set -x
mkdir -p gpurun_out
for lib in b512m2 b1024m1 mb3; do
  if [ $lib = base ]; then unset MFX_LIB_PATH; else export MFX_LIB_PATH=$PWD/build/$lib/libmfx.so; fi
  timeout 300 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 4 --barrier --knobs '' > gpurun_out/mb_${lib}_C2.log 2>&1
  timeout 300 python scripts/sweep.py --graph rmat --scale 20 --batch 10000 --batches 3 --knobs '' > gpurun_out/mb_${lib}_C3.log 2>&1
  timeout 300 python scripts/sweep.py --graph road --side 1024 --batch 10000 --batches 2 --knobs '' > gpurun_out/mb_${lib}_road.log 2>&1
done
for f in gpurun_out/mb_*.log; do echo -n "$(basename $f) "; python scripts/sweep_table.py $f | grep default | cut -c30-200; done
