mkdir -p gpurun_out
for i in 1 2 3; do
MFX_TIMEOUT_S=20 timeout 400 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/dbg$i.log 2>&1
tail -30 gpurun_out/dbg$i.log | grep -v "^\.\.\." | tail -25
done
