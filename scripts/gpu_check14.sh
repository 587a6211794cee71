set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-300
for g in "grid --side 2048 --batch 10000 --batches 4" "rmat --scale 20 --batch 10000 --batches 3" "road --side 1024 --batch 10000 --batches 2" "random --batch 1000 --batches 3"; do
  name=$(echo $g | cut -d' ' -f1-3 | tr ' ' '_')
  timeout 300 python scripts/sweep.py --graph $g --knobs '' > gpurun_out/c14_${name}.log 2>&1
done
MFX_TIMEOUT_S=300 timeout 900 python scripts/sweep.py --graph road --side 4900 --batch 10000 --batches 2 --knobs '' > gpurun_out/c14_C4.log 2>&1
MFX_TRACE_CAP=400000 timeout 300 python scripts/trace.py --side 2048 > gpurun_out/trace_C2.log 2>&1
