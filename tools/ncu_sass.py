"""Dev helper: summarise an ncu report's SASS hot spots (not part of the product).

    python tools/ncu_sass.py REPORT [N]            top-N stalled instructions
    python tools/ncu_sass.py REPORT --at ADDR [B] [A]   context around an address suffix
"""
import csv
import subprocess
import sys


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout.splitlines()
    r = list(csv.reader(out[1:]))
    h = r[0]
    return h, r[1:]


def main():
    rep = sys.argv[1]
    h, rs = rows(rep)
    ia, isrc, iall = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    if len(sys.argv) > 2 and sys.argv[2] == "--at":
        suf = sys.argv[3]
        b = int(sys.argv[4]) if len(sys.argv) > 4 else 12
        a = int(sys.argv[5]) if len(sys.argv) > 5 else 4
        for k, r in enumerate(rs):
            if len(r) > ia and r[ia].endswith(suf):
                for rr in rs[max(0, k - b):k + a]:
                    print(f"{rr[iall]:>7} {rr[ia][-5:]} {rr[isrc].strip()}")
        return
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    data, tot = [], 0
    for r in rs:
        try:
            s = int(r[iall])
        except Exception:
            continue
        tot += s
        data.append((s, r[ia], r[isrc]))
    data.sort(reverse=True)
    print("total samples", tot)
    for s, a, src in data[:n]:
        print(f"{s:7d} {100 * s / tot:5.1f}%  {a[-5:]}  {src.strip()}")


if __name__ == "__main__":
    main()
