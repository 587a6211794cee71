"""Compact table of scripts/sweep.py JSON lines: python scripts/sweep_table.py LOG..."""
import json
import sys

for path in sys.argv[1:]:
    print("##", path)
    for line in open(path):
        if line.startswith("{"):
            d = json.loads(line)
            print(f"{d['knobs']:28s} static {d['static_ms']:8.2f} (bfs {d['st_bfs_ms']:6.2f} push "
                  f"{d['st_push_ms']:6.2f} ep {d.get('st_epochs')}) | dyn {d['dyn_ms']:7.2f} (bfs "
                  f"{d['dyn_bfs_ms']:6.2f} push {d['dyn_push_ms']:6.2f} ep {d.get('dyn_epochs')} "
                  f"rounds {d['dyn_rounds']} waves {d['dyn_waves']}) ok={d['flows_agree']}")
        elif line.startswith("#"):
            print(line.strip()[:110])
