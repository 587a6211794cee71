bash scripts/gpu_sanitize.sh > /dev/null 2>&1
bash scripts/gpu_racecheck.sh > /dev/null 2>&1
for f in memcheck memcheck2 racecheck synccheck; do echo "== $f"; tail -6 gpurun_out/$f.log; done
