for r in 1 2; do
  echo "== 0e0cfac"; (cd abl/0e0cfac && python c4_probe.py --graph grid --side 2048 --batches 10 --quiet | grep "#")
  echo "== HEAD"; python scripts/c4_probe.py --graph grid --side 2048 --batches 10 --quiet | grep "#"
done
python scripts/static_ab.py --graph grid --side 2048 --reps 3 --knobs ""
python scripts/c4_probe.py --batches 30 --quiet | grep "#"
python scripts/c4_probe.py --graph rmat --side 20 --batches 6 --quiet | grep "#"
python scripts/static_ab.py --graph rmat --side 20 --reps 3 --knobs ""
