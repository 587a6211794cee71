set -x
mkdir -p gpurun_out
for wm in "0 0" "100000000 0" "4096 0" "100000000 256" "100000000 1024"; do
 set -- $wm
 for g in "grid --side 2048 --batch 10000 --batches 4" "rmat --scale 20 --batch 10000 --batches 3" "road --side 1024 --batch 10000 --batches 2" "random --batch 1000 --batches 3"; do
  name=$(echo $g | cut -d' ' -f1)
  MFX_WALK_MAX=$1 MFX_WALK_DEPTH=$2 timeout 300 python scripts/sweep.py --graph $g --knobs '' > gpurun_out/walk_${name}_$1_$2.log 2>&1
 done
done
for f in gpurun_out/walk_*.log; do echo -n "$(basename $f) "; python scripts/sweep_table.py $f | grep default | cut -c30-200; done
MFX_WALK_MAX=100000000 timeout 900 python -m pytest tests -m gpu -x -q -k "flows or large or random_vs_oracle or pushpull or instrument" > gpurun_out/pytest_walk.log 2>&1; tail -3 gpurun_out/pytest_walk.log
