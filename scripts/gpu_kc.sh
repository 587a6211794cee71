set -x
mkdir -p gpurun_out
K="'' kernel_cycles=1 kernel_cycles=2 kernel_cycles=10 kernel_cycles=32"
eval timeout 300 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 4 --knobs $K > gpurun_out/kc_grid.log 2>&1
eval timeout 300 python scripts/sweep.py --graph rmat --scale 20 --batch 10000 --batches 3 --knobs $K > gpurun_out/kc_rmat.log 2>&1
eval timeout 300 python scripts/sweep.py --graph road --side 1024 --batch 10000 --batches 2 --knobs $K > gpurun_out/kc_road.log 2>&1
python scripts/sweep_table.py gpurun_out/kc_*.log
