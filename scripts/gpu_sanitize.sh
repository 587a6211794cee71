# compute-sanitizer memcheck / racecheck-lite on small graphs (race detection)
set -x
mkdir -p gpurun_out
export MFX_TIMEOUT_S=120
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 17 python -m pytest tests/test_gpu_parity.py -x -q -k "rand0 or rand3 or diamond or grid64 or edge_cases or wide" > gpurun_out/memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/memcheck.log; tail -5 gpurun_out/memcheck.log
timeout 1200 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 17 python -m pytest tests/test_gpu_partition.py tests/test_gpu_pushpull.py -x -q -k "rand3 or rand0 or errors or certificate" > gpurun_out/memcheck2.log 2>&1; echo "memcheck2 rc=$?" >> gpurun_out/memcheck2.log; tail -5 gpurun_out/memcheck2.log
