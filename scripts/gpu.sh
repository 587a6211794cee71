# One parameterised gpurun recipe (replaces the round-1 per-experiment scripts).
#
#   gpurun --timeout 1800 -- 'bash scripts/gpu.sh tests smoke bench'
#   gpurun -- 'bash scripts/gpu.sh "sweep:road --side 4900 --batch 10000 --batches 4 --knobs \"\" MFX_X=1"'
#   gpurun -- 'bash scripts/gpu.sh "bench:--config C2 --steps 10" ncu_c4 launches_c4'
#
# Every task writes gpurun_out/<task>.log and prints its tail.  Tasks:
#   tests            pytest -m gpu (the driver's round-end suite)
#   slow             pytest -m "gpu and slow" (opt-in large partition / stress tests)
#   smoke            __graft_entry__.smoke()
#   bench[:ARGS]     python bench.py ARGS (default: the C4 headline)
#   ref[:ARGS]       python bench.py --impl reference ARGS
#   sweep:ARGS       python scripts/sweep.py ARGS
#   ncu_<cfg>        ncu --set full of the first timed solve_kernel launch of bench.py --profile
#                    (NVTX range "timed") -> .ncu-rep (summarise here: scripts/ncu_summary.py)
#   launches_<cfg>   ncu launch list (gpu__time_duration.sum) of bench.py --profile
#   sanitize         compute-sanitizer memcheck + synccheck over the parity tests
#   cmd:SHELL        any shell command
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv,noheader
i=0
for task in "$@"; do
  i=$((i + 1))
  name="${task%%:*}"
  args=""
  [ "$name" != "$task" ] && args="${task#*:}"
  log="gpurun_out/${i}_${name}.log"
  case "$name" in
    tests)    timeout 1500 python -m pytest tests -m gpu -x -q $args > "$log" 2>&1 ;;
    slow)     timeout 2400 python -m pytest tests -m "gpu and slow" -x -q $args > "$log" 2>&1 ;;
    smoke)    timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$log" 2>&1 ;;
    bench)    eval "timeout 1200 python bench.py $args" > "$log" 2>&1 ;;
    ref)      eval "timeout 1500 python bench.py --impl reference $args" > "$log" 2>&1 ;;
    sweep)    eval "MFX_TIMEOUT_S=300 timeout 1500 python scripts/sweep.py $args" > "$log" 2>&1 ;;
    ncu_*)    cfg=$(echo "${name#ncu_}" | tr a-z A-Z)
              timeout 1500 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" \
                -k regex:^solve_kernel -c 1 -f -o gpurun_out/prof_${cfg}_dyn \
                python bench.py --config $cfg --profile --steps 1 --warmup 3 $args > "$log" 2>&1 ;;
    launches_*) cfg=$(echo "${name#launches_}" | tr a-z A-Z)
              timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
                --log-file gpurun_out/launches_${cfg}.csv python bench.py --config $cfg --profile --steps 3 --warmup 3 $args > "$log" 2>&1 ;;
    sanitize) timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest -x -q -m gpu \
                tests/test_gpu_parity.py -k "bit_exact or random" > "$log" 2>&1
              timeout 2400 compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest -x -q -m gpu \
                tests/test_gpu_parity.py -k "bit_exact" >> "$log" 2>&1 ;;
    cmd)      eval "$args" > "$log" 2>&1 ;;
    *)        echo "unknown task $name" > "$log" ;;
  esac
  echo "== $task rc=$?"
  tail -4 "$log" | cut -c1-1500
done
