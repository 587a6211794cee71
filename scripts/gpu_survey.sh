# Round-1 GPU survey: per-config timing, phase trace, ncu launch list + full capture.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 300 python scripts/sweep.py --graph random --batch 1000 --batches 3 --knobs '' 'schedule=async' > gpurun_out/sweep_C1.log 2>&1
timeout 300 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 3 --barrier --knobs '' 'schedule=async' 'max_waves=1' > gpurun_out/sweep_C2.log 2>&1
timeout 300 python scripts/sweep.py --graph rmat --scale 20 --batch 10000 --batches 3 --knobs '' 'schedule=async' > gpurun_out/sweep_C3.log 2>&1
timeout 300 python scripts/sweep.py --graph rmat --scale 20 --batch 100000 --batches 2 --knobs '' > gpurun_out/sweep_C3_100k.log 2>&1
timeout 300 python scripts/sweep.py --graph road --side 1024 --batch 10000 --batches 2 --knobs '' 'schedule=async' > gpurun_out/sweep_road1024.log 2>&1
MFX_TIMEOUT_S=200 timeout 900 python scripts/sweep.py --graph road --side 4900 --batch 10000 --batches 2 --knobs 'schedule=async' > gpurun_out/sweep_C4.log 2>&1
MFX_TRACE_CAP=400000 timeout 300 python scripts/trace.py --side 2048 > gpurun_out/trace_C2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2.csv python bench.py --profile --steps 3 --warmup 3 > gpurun_out/launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:solve_kernel -s 2 -c 1 -o gpurun_out/prof_C2_dyn python scripts/profile_target.py --batches 1 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
