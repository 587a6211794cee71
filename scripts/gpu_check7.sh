set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pushpull.py -x -q > gpurun_out/pytest_pp.log 2>&1; tail -3 gpurun_out/pytest_pp.log
timeout 400 python scripts/sweep.py --graph grid --side 2048 --batch 10000 --batches 4 --knobs '' 'pp=1' > gpurun_out/sw9_C2.log 2>&1
timeout 300 python scripts/sweep.py --graph rmat --scale 20 --batch 10000 --batches 3 --knobs '' 'pp=1' > gpurun_out/sw9_C3.log 2>&1
python scripts/sweep_table.py gpurun_out/sw9_*.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
