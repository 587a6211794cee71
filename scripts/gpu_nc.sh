set -x
mkdir -p gpurun_out
for g in "grid --side 2048 --batch 10000 --batches 4" "rmat --scale 20 --batch 10000 --batches 3" "road --side 1024 --batch 10000 --batches 2" "random --batch 1000 --batches 3"; do
  name=$(echo $g | cut -d' ' -f1)
  timeout 300 python scripts/sweep.py --graph $g --knobs '' 'device_flags=2' > gpurun_out/nc_${name}.log 2>&1
done
python scripts/sweep_table.py gpurun_out/nc_*.log
