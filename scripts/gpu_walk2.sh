set -x
mkdir -p gpurun_out
for wm in "-1 0" "32 1" "256 1" "2048 1"; do
 set -- $wm
 MFX_WALK_MAX=$1 MFX_WALK_DEPTH=$2 timeout 300 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 6 --knobs '' > gpurun_out/walk2_grid_$1_$2.log 2>&1
 MFX_WALK_MAX=$1 MFX_WALK_DEPTH=$2 timeout 300 python scripts/sweep.py --graph random --batch 1000 --batches 6 --knobs '' > gpurun_out/walk2_random_$1_$2.log 2>&1
done
for f in gpurun_out/walk2_*.log; do echo -n "$(basename $f) "; python scripts/sweep_table.py $f | grep default | cut -c30-200; done
