set -x
mkdir -p gpurun_out
for mc in 0 148; do
  MFX_MAX_CTAS=$mc timeout 300 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 4 --knobs '' > gpurun_out/ctas2_grid_$mc.log 2>&1
  MFX_MAX_CTAS=$mc timeout 300 python scripts/sweep.py --graph rmat --scale 20 --batch 10000 --batches 3 --knobs '' > gpurun_out/ctas2_rmat_$mc.log 2>&1
  MFX_MAX_CTAS=$mc timeout 300 python scripts/sweep.py --graph road --side 1024 --batch 10000 --batches 2 --knobs '' > gpurun_out/ctas2_road_$mc.log 2>&1
done
for f in gpurun_out/ctas2_*.log; do echo -n "$(basename $f) "; python scripts/sweep_table.py $f | grep default | cut -c30-200; done
