set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
MFX_FLAGS=8 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -m gpu -x -q -k "flows or bit_exact" > gpurun_out/pytest_retry.log 2>&1; tail -3 gpurun_out/pytest_retry.log
for g in "grid --side 2048 --batch 10000 --batches 4" "road --side 1024 --batch 10000 --batches 2"; do
  name=$(echo $g | cut -d' ' -f1)
  timeout 300 python scripts/sweep.py --graph $g --knobs '' > gpurun_out/sw15_${name}.log 2>&1
done
for f in gpurun_out/sw15_*.log; do echo -n "$(basename $f) "; python scripts/sweep_table.py $f | grep default | cut -c30-200; done
