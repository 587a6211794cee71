set -x
mkdir -p gpurun_out
for lib in old new; do
  if [ $lib = old ]; then export MFX_LIB_PATH=$PWD/build/old/libmfx.so; else unset MFX_LIB_PATH; fi
  timeout 300 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 3 --knobs '' 'bfs_local=-1' 'bfs_local=8' 'bfs_local=32' > gpurun_out/ab_${lib}_C2.log 2>&1
  timeout 300 python scripts/sweep.py --graph road --side 1024 --batch 10000 --batches 2 --knobs '' 'bfs_local=-1' 'bfs_local=32' 'bfs_local=128' > gpurun_out/ab_${lib}_road.log 2>&1
done
for f in gpurun_out/ab_*.log; do echo "## $f"; cut -c1-330 $f; done
