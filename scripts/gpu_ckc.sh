set -x
mkdir -p gpurun_out
for ck in 0 1 2; do
 for g in "grid --side 2048 --batch 10000 --batches 4" "rmat --scale 20 --batch 10000 --batches 3" "road --side 1024 --batch 10000 --batches 2" "random --batch 1000 --batches 3"; do
  name=$(echo $g | cut -d' ' -f1)
  MFX_COOP_KC=$ck timeout 300 python scripts/sweep.py --graph $g --knobs '' 'kernel_cycles=2' > gpurun_out/ckc_${name}_${ck}.log 2>&1
 done
done
for f in gpurun_out/ckc_*.log; do echo "$(basename $f)"; python scripts/sweep_table.py $f | grep -v "^#" | cut -c1-200; done
