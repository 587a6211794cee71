set -x
mkdir -p gpurun_out
for lib in base wq128; do
  if [ $lib = base ]; then unset MFX_LIB_PATH; else export MFX_LIB_PATH=$PWD/build/$lib/libmfx.so; fi
  for g in "grid --side 2048 --batch 10000 --batches 4" "rmat --scale 20 --batch 10000 --batches 3" "road --side 1024 --batch 10000 --batches 2" "random --batch 1000 --batches 3"; do
    name=$(echo $g | cut -d' ' -f1)
    timeout 300 python scripts/sweep.py --graph $g --knobs '' > gpurun_out/wq_${lib}_${name}.log 2>&1
  done
done
for f in gpurun_out/wq_*.log; do echo -n "$(basename $f) "; python scripts/sweep_table.py $f | grep default | cut -c30-200; done
