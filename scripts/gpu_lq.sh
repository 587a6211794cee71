set -x
mkdir -p gpurun_out
for cap in 2048 1024 512 256; do
  for lm in 64 256; do
    echo "== lq_cap=$cap bfs_local_max=$lm"
    MFX_LQ_CAP=$cap MFX_BFS_LOCAL_MAX=$lm timeout 300 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 4 --knobs '' > gpurun_out/lq_C2_${cap}_${lm}.log 2>&1
    MFX_LQ_CAP=$cap MFX_BFS_LOCAL_MAX=$lm timeout 300 python scripts/sweep.py --graph road --side 1024 --batch 10000 --batches 2 --knobs '' > gpurun_out/lq_road_${cap}_${lm}.log 2>&1
  done
done
for f in gpurun_out/lq_*.log; do echo $f; python scripts/sweep_table.py $f | tail -2 | head -1; done
