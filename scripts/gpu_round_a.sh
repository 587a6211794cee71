set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-1600
MFX_TIMEOUT_S=300 timeout 900 python scripts/sweep.py --graph road --side 4900 --batch 10000 --batches 2 --knobs '' > gpurun_out/sweep_C4.log 2>&1; python scripts/sweep_table.py gpurun_out/sweep_C4.log
timeout 600 python bench.py --config C5 --steps 3 --warmup 1 > gpurun_out/bench_c5.log 2>&1; tail -1 gpurun_out/bench_c5.log | cut -c1-1500
timeout 900 ncu --set full --clock-control none --import-source on -k solve_kernel -s 2 -c 1 -o gpurun_out/prof_C2_dyn python scripts/profile_target.py --batches 1 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2.csv python bench.py --profile --steps 3 --warmup 3 > gpurun_out/launches_bench.log 2>&1
