for c in b8fac0c acb8ce1 0e0cfac 53e2982; do echo "== $c"; (cd abl/$c && python static_ab.py --graph grid --side 2048 --knobs "" 2>&1 | tail -1); done
echo "== HEAD"; python scripts/static_ab.py --graph grid --side 2048 --knobs "" 2>&1 | tail -1
