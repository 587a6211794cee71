# Round-end evidence: full GPU suite, smoke, headline bench, C5 bench, sweeps, ncu.
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-300
timeout 900 python bench.py --config C5 --steps 3 --warmup 1 > gpurun_out/bench_c5.log 2>&1; tail -1 gpurun_out/bench_c5.log | cut -c1-300
for g in "grid --side 2048 --batch 10000 --batches 4" "rmat --scale 20 --batch 10000 --batches 3" "rmat --scale 20 --batch 100000 --batches 2" "road --side 1024 --batch 10000 --batches 2" "random --batch 1000 --batches 3"; do
  name=$(echo $g | cut -d' ' -f1-5 | tr ' ' '_')
  timeout 300 python scripts/sweep.py --graph $g --knobs '' 'pp=1' > gpurun_out/final_${name}.log 2>&1
done
MFX_TIMEOUT_S=300 timeout 900 python scripts/sweep.py --graph road --side 4900 --batch 10000 --batches 2 --knobs '' > gpurun_out/final_C4.log 2>&1
for f in gpurun_out/final_*.log; do echo "$(basename $f)"; python scripts/sweep_table.py $f | grep -v "^#"; done
timeout 900 ncu --set full --clock-control none --import-source on -k solve_kernel -s 2 -c 1 -o gpurun_out/prof_C2_dyn python scripts/profile_target.py --batches 1 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2.csv python bench.py --profile --steps 3 --warmup 3 > gpurun_out/launches_bench.log 2>&1
MFX_TRACE_CAP=400000 timeout 300 python scripts/trace.py --side 2048 > gpurun_out/trace_C2.log 2>&1
