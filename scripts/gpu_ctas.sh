set -x
mkdir -p gpurun_out
for mc in 0 148 64 32 16; do
  MFX_MAX_CTAS=$mc timeout 300 python scripts/sweep.py --graph random --batch 1000 --batches 6 --barrier --knobs '' > gpurun_out/ctas_random_$mc.log 2>&1
done
for mc in 0 148; do
  MFX_MAX_CTAS=$mc timeout 300 python scripts/sweep.py --graph grid --side 512 --batch 10000 --batches 4 --knobs '' > gpurun_out/ctas_grid512_$mc.log 2>&1
  MFX_MAX_CTAS=$mc timeout 300 python scripts/sweep.py --graph rmat --scale 16 --batch 1000 --batches 4 --knobs '' > gpurun_out/ctas_rmat16_$mc.log 2>&1
done
for f in gpurun_out/ctas_*.log; do echo -n "$(basename $f) "; python scripts/sweep_table.py $f | grep default | cut -c30-200; done
