set -x
mkdir -p gpurun_out
for g in "grid --side 2048 --batch 10000 --batches 4" "rmat --scale 20 --batch 10000 --batches 3" "road --side 1024 --batch 10000 --batches 2" "random --batch 1000 --batches 3"; do
  name=$(echo $g | cut -d' ' -f1)
  timeout 300 python scripts/sweep.py --graph $g --knobs '' 'device_flags=4' > gpurun_out/early_${name}.log 2>&1
done
python scripts/sweep_table.py gpurun_out/early_*.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
MFX_TRACE_CAP=400000 timeout 300 python scripts/trace.py --side 2048 > gpurun_out/trace_C2.log 2>&1; grep -A10 "per-round" gpurun_out/trace_C2.log
