python scripts/static_ab.py --graph rmat --side 20 --reps 3 --knobs "" MFX_BU_DIV=0
python scripts/c4_probe.py --graph rmat --side 20 --batch 10000 --batches 6 --quiet --knobs "" MFX_BU_DIV=0 | grep "#"
python scripts/c4_probe.py --graph rmat --side 20 --batch 100000 --batches 4 --quiet --knobs "" MFX_BU_DIV=0 | grep "#"
python scripts/static_ab.py --graph grid --side 2048 --reps 3 --knobs "" MFX_BU_DIV=0
python scripts/c4_probe.py --graph grid --side 2048 --batches 10 --quiet --knobs "" MFX_BU_DIV=0 | grep "#"
python scripts/c4_probe.py --graph random --batch 1000 --batches 10 --quiet --knobs "" MFX_BU_DIV=0 | grep "#"
python scripts/c4_probe.py --batches 20 --quiet | grep "#"
