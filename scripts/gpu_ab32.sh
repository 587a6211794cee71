set -x
mkdir -p gpurun_out
K="'' MFX_BFS_LOCAL=-1 MFX_BFS_LOCAL=4 MFX_BFS_LOCAL_MAX=8"
for rep in 1 2; do
eval timeout 400 python scripts/sweep.py --graph random --batch 1000 --batches 6 --knobs $K > gpurun_out/ab32_${rep}_C1.log 2>&1
done
