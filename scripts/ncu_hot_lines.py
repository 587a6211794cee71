"""Aggregate warp-stall samples per CUDA source line from an ncu report
(ncu -i X.ncu-rep --page source --csv --print-source cuda,sass).

    python scripts/ncu_hot_lines.py gpurun_out/prof.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname = None
    agg = {}
    total = 0
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if len(r) < 6 or r[0] == "Line No" or r[2] != "-":
            continue  # only CUDA-line rows (SASS rows carry an address in col 2)
        try:
            s = int(r[4])
        except ValueError:
            continue
        total += s
        agg[(fname, int(r[0]))] = (agg.get((fname, int(r[0])), (0, ""))[0] + s, r[1].strip()[:90])
    print(f"total warp-stall samples: {total}")
    for (f, ln), (s, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{100 * s / max(total, 1):5.1f}%  {f}:{ln:<5d} {src}")


if __name__ == "__main__":
    main()
