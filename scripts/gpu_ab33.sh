set -x
mkdir -p gpurun_out
K="'' MFX_BFS_LOCAL=-1"
for rep in 1 2; do
eval timeout 400 python scripts/sweep.py --graph rmat --scale 20 --batch 10000 --batches 4 --knobs $K pp=1 pp=1,MFX_BFS_LOCAL=-1 > gpurun_out/ab33_${rep}_C3.log 2>&1
eval timeout 400 python scripts/sweep.py --graph rmat --scale 18 --batch 10000 --batches 4 --knobs $K > gpurun_out/ab33_${rep}_r18.log 2>&1
done
