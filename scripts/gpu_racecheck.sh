set -x
mkdir -p gpurun_out
export MFX_TIMEOUT_S=300
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard python -m pytest tests/test_gpu_parity.py -x -q -k "rand0 or diamond" > gpurun_out/racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/racecheck.log; tail -15 gpurun_out/racecheck.log
timeout 900 compute-sanitizer --tool synccheck python -m pytest tests/test_gpu_parity.py -x -q -k "rand0 or diamond" > gpurun_out/synccheck.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/synccheck.log; tail -8 gpurun_out/synccheck.log
