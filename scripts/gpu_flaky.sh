mkdir -p gpurun_out
for i in 1 2 3; do
  timeout 900 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/flaky_$i.log 2>&1; tail -1 gpurun_out/flaky_$i.log
done
