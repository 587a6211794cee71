#!/bin/bash
# Build libmfx.so + oracle and fail loudly if anything is stale or broken.
set -e
cd "$(dirname "$0")/.."
make -s -j4 -C paper_2511_01235_b200/csrc
make -s -C oracle
lib=paper_2511_01235_b200/_lib/libmfx.so
for f in paper_2511_01235_b200/csrc/*.cu paper_2511_01235_b200/csrc/*.h paper_2511_01235_b200/csrc/*.cuh include/mfx.h; do
  if [ "$f" -nt "$lib" ]; then echo "STALE: $f newer than $lib"; exit 1; fi
done
grep -h -A3 "solve_kernelI" paper_2511_01235_b200/_lib/obj/solve.ptxas.log | grep -E "registers|spill" || true
echo "build ok"
