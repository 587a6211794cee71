for r in 1 2; do
  echo "== 0e0cfac"; (cd abl/0e0cfac && python c4_probe.py --graph grid --side 2048 --batches 10 --quiet | grep "#")
  for c in 53e2982 58a40aa f819148 0d08b32; do
    echo "== $c"; (cd abl/$c && python scripts/c4_probe.py --graph grid --side 2048 --batches 10 --quiet | grep "#")
  done
  echo "== HEAD"; python scripts/c4_probe.py --graph grid --side 2048 --batches 10 --quiet | grep "#"
done
