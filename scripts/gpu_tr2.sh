mkdir -p gpurun_out
MFX_TRACE_CAP=400000 timeout 300 python scripts/trace.py --side 2048 > gpurun_out/trace_C2.log 2>&1
