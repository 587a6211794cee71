# ncu of the global relabel alone (WHAT_BFS launch on the state after one C2 batch)
set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k solve_kernel -s 5 -c 1 -o gpurun_out/prof_C2_bfs python scripts/profile_target.py --batches 1 --relabels 4 > gpurun_out/ncu_bfs.log 2>&1
tail -3 gpurun_out/ncu_bfs.log
MFX_TRACE_CAP=10000 timeout 300 python scripts/profile_target.py --batches 1 --relabels 4 > gpurun_out/bfs_plain.log 2>&1
