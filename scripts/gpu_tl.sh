set -x
mkdir -p gpurun_out
for tl in 0 256 2048; do
 for g in "grid --side 2048 --batch 10000 --batches 4" "rmat --scale 20 --batch 10000 --batches 3" "road --side 1024 --batch 10000 --batches 2" "random --batch 1000 --batches 4"; do
  name=$(echo $g | cut -d' ' -f1)
  MFX_TAIL_LOCAL=$tl timeout 300 python scripts/sweep.py --graph $g --knobs '' > gpurun_out/tl_${name}_${tl}.log 2>&1
 done
done
for f in gpurun_out/tl_*.log; do echo -n "$(basename $f) "; python scripts/sweep_table.py $f | grep default | cut -c30-200; done
MFX_TAIL_LOCAL=2048 timeout 900 python -m pytest tests -m gpu -x -q -k "flows or large or random_vs_oracle or pushpull or instrument or c4" > gpurun_out/pytest_tl.log 2>&1; tail -3 gpurun_out/pytest_tl.log
