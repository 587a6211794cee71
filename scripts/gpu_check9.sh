set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for g in "grid --side 2048 --batch 10000 --batches 4" "rmat --scale 20 --batch 10000 --batches 3" "road --side 1024 --batch 10000 --batches 2" "random --batch 1000 --batches 3"; do
  name=$(echo $g | cut -d' ' -f1)
  timeout 300 python scripts/sweep.py --graph $g --knobs '' > gpurun_out/sw11_${name}.log 2>&1
  MFX_VARIANT=512 timeout 300 python scripts/sweep.py --graph $g --knobs '' > gpurun_out/sw11_${name}_v512.log 2>&1
  MFX_VARIANT=256 timeout 300 python scripts/sweep.py --graph $g --knobs '' > gpurun_out/sw11_${name}_v256.log 2>&1
done
for f in gpurun_out/sw11_*.log; do echo -n "$(basename $f) "; python scripts/sweep_table.py $f | grep default | cut -c30-200; done
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-400
