mkdir -p gpurun_out
for lib in old new; do
  if [ $lib = old ]; then export MFX_LIB_PATH=$PWD/build/old/libmfx.so; else unset MFX_LIB_PATH; fi
  echo "== $lib"; timeout 300 python scripts/repair_probe.py 2048
done > gpurun_out/rp.log 2>&1
cat gpurun_out/rp.log
