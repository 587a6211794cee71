set -x
mkdir -p gpurun_out
K="'' wave_mult=4,wave_add=16 wave_mult=8,wave_add=64 max_waves=2000 bfs_local=8 bfs_local=128"
for lib in base b512; do
  if [ $lib = b512 ]; then export MFX_LIB_PATH=$PWD/build/b512/libmfx.so; else unset MFX_LIB_PATH; fi
  eval timeout 400 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 4 --barrier --knobs $K > gpurun_out/sw2_${lib}_C2.log 2>&1
  eval timeout 300 python scripts/sweep.py --graph rmat --scale 20 --batch 10000 --batches 3 --knobs $K > gpurun_out/sw2_${lib}_C3.log 2>&1
  eval timeout 300 python scripts/sweep.py --graph road --side 1024 --batch 10000 --batches 2 --knobs "''" bfs_local=128 > gpurun_out/sw2_${lib}_road.log 2>&1
done
