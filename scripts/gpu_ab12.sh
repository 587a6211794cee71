set -x
mkdir -p gpurun_out
for rep in 1 2; do
  timeout 400 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 4 --knobs '' > gpurun_out/ab12_${rep}_C2.log 2>&1
  MFX_VARIANT=512 timeout 400 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 4 --knobs '' > gpurun_out/ab12_${rep}_C2_512.log 2>&1
  MFX_VARIANT=512 timeout 400 python scripts/sweep.py --graph road --side 1024 --batch 10000 --batches 2 --knobs '' > gpurun_out/ab12_${rep}_road_512.log 2>&1
done
