mkdir -p gpurun_out
for g in grid64 rmat12 rand3; do echo "== $g"; timeout 120 python scripts/bfs_probe.py $g; done > gpurun_out/bp.log 2>&1
cat gpurun_out/bp.log
