"""Dev helper: per-CUDA-source-line totals (stall samples, executed warp
instructions) from an ncu report captured with --import-source on.

    python tools/ncu_lines.py REPORT [N] [FILE_SUBSTR]
"""
import csv
import subprocess
import sys
from collections import defaultdict


def main():
    rep = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    filt = sys.argv[3] if len(sys.argv) > 3 else ""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout.splitlines()
    rows = list(csv.reader(out))
    path = ""
    stall = defaultdict(float)
    inst = defaultdict(float)
    text = {}
    hdr = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            path = r[1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0].isdigit():
            continue
        if filt and filt not in path:
            continue
        key = (path.split("/")[-1], int(r[0]))
        text[key] = r[1]
        try:
            stall[key] += float(r[4] or 0)
            inst[key] += float(r[7] or 0)
        except (ValueError, IndexError):
            pass
    tot_s = sum(stall.values()) or 1
    tot_i = sum(inst.values()) or 1
    print(f"samples {tot_s:.0f}  warp-inst {tot_i:.3e}")
    for key in sorted(stall, key=lambda k: -stall[k])[:n]:
        print(f"{100*stall[key]/tot_s:5.1f}% {100*inst[key]/tot_i:5.1f}%i  "
              f"{key[0]}:{key[1]:<5} {text[key].strip()[:90]}")


if __name__ == "__main__":
    main()
