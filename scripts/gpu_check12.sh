set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for g in "grid --side 2048 --batch 10000 --batches 6" "rmat --scale 20 --batch 10000 --batches 3" "road --side 1024 --batch 10000 --batches 2" "random --batch 1000 --batches 4"; do
  name=$(echo $g | cut -d' ' -f1)
  timeout 300 python scripts/sweep.py --graph $g --knobs '' > gpurun_out/sw14_${name}.log 2>&1
done
for f in gpurun_out/sw14_*.log; do echo -n "$(basename $f) "; python scripts/sweep_table.py $f | grep default | cut -c30-200; done
