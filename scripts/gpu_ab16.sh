set -x
mkdir -p gpurun_out
K="'' wave_mult=1,wave_add=4 wave_mult=1,wave_add=16 wave_mult=3,wave_add=4 max_waves=16 max_waves=32"
eval timeout 400 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 4 --knobs $K > gpurun_out/ab16_C2.log 2>&1
eval timeout 400 python scripts/sweep.py --graph road --side 1024 --batch 10000 --batches 2 --knobs $K > gpurun_out/ab16_road.log 2>&1
eval timeout 400 python scripts/sweep.py --graph rmat --scale 20 --batch 10000 --batches 4 --knobs $K > gpurun_out/ab16_C3.log 2>&1
eval timeout 400 python scripts/sweep.py --graph random --batch 1000 --batches 6 --knobs $K > gpurun_out/ab16_C1.log 2>&1
