"""Summarise an ncu report: top stalled SASS instructions and stall reasons (dev helper)."""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
h = rows[0]
ia, isrc, iall = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
data = []
tot = 0
for r in rows[1:]:
    try:
        s = int(r[iall])
    except Exception:
        continue
    tot += s
    data.append((s, r[ia], r[isrc]))
data.sort(reverse=True)
print("total samples", tot)
for s, a, src in data[:n]:
    print(f"{s:7d} {100*s/tot:5.1f}%  {a[-5:]}  {src.strip()}")
