set -x
mkdir -p gpurun_out
for ti in 0 256 1024 4096; do
 for tc in 200 1000; do
  for g in "grid --side 2048 --batch 10000 --batches 4" "rmat --scale 20 --batch 10000 --batches 3" "road --side 1024 --batch 10000 --batches 2" "random --batch 1000 --batches 3"; do
    name=$(echo $g | cut -d' ' -f1)
    MFX_TAIL_ITEMS=$ti MFX_TAIL_CAP=$tc timeout 300 python scripts/sweep.py --graph $g --knobs '' > gpurun_out/tail_${name}_${ti}_${tc}.log 2>&1
  done
 done
done
for f in gpurun_out/tail_*.log; do echo -n "$(basename $f) "; python scripts/sweep_table.py $f | grep default | cut -c30-200; done
