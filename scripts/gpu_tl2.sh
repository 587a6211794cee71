set -x
mkdir -p gpurun_out
for tl in 0 256; do
 for g in "grid --side 2048 --batch 10000 --batches 4" "road --side 1024 --batch 10000 --batches 2" "random --batch 1000 --batches 4" "grid --side 512 --batch 10000 --batches 4"; do
  name=$(echo $g | cut -d' ' -f1-3 | tr ' ' '_')
  MFX_TAIL_LOCAL=$tl timeout 300 python scripts/sweep.py --graph $g --knobs '' > gpurun_out/tl2_${name}_${tl}.log 2>&1
 done
done
MFX_TIMEOUT_S=300 timeout 900 python scripts/sweep.py --graph road --side 4900 --batch 10000 --batches 2 --knobs '' > gpurun_out/tl2_C4.log 2>&1
for f in gpurun_out/tl2_*.log; do echo -n "$(basename $f) "; python scripts/sweep_table.py $f | grep default | cut -c30-200; done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
