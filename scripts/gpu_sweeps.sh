# The sweep part of gpu_final.sh (configs C1-C4 + push-pull)
mkdir -p gpurun_out
for g in "grid --side 2048 --batch 10000 --batches 4" "rmat --scale 20 --batch 10000 --batches 3" "rmat --scale 20 --batch 100000 --batches 2" "road --side 1024 --batch 10000 --batches 2" "random --batch 1000 --batches 3"; do
  name=$(echo $g | cut -d' ' -f1-5 | tr ' ' '_')
  timeout 300 python scripts/sweep.py --graph $g --knobs '' 'pp=1' > gpurun_out/final_${name}.log 2>&1
done
MFX_TIMEOUT_S=300 timeout 900 python scripts/sweep.py --graph road --side 4900 --batch 10000 --batches 2 --knobs '' > gpurun_out/final_C4.log 2>&1
