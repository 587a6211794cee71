# ncu evidence for the persistent solve kernel (C2 dynamic batch 1) + clean bench line.
set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k solve_kernel -s 2 -c 1 -o gpurun_out/prof_C2_dyn python scripts/profile_target.py --batches 1 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k solve_kernel -s 1 -c 1 -o gpurun_out/prof_C2_static python scripts/profile_target.py --batches 0 > gpurun_out/ncu_full_static.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
tail -2 gpurun_out/ncu_full.log
