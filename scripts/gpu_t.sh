mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k schedule > gpurun_out/pt.log 2>&1; tail -5 gpurun_out/pt.log
