"""Summarise sweep.py logs: one line per knob setting."""
import json
import sys

for path in sys.argv[1:]:
    print("##", path)
    for line in open(path):
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        print("%-24s st %8.2f dyn %7.2f stbfs %7.2f dynbfs %6.2f stpush %7.2f dynpush %6.2f ep %s/%s ok %s"
              % (d["knobs"], d["static_ms"], d["dyn_ms"], d["st_bfs_ms"], d["dyn_bfs_ms"],
                 d["st_push_ms"], d["dyn_push_ms"], d["st_epochs"], d["dyn_epochs"], d["flows_agree"]))
