"""Dev helper: DRAM traffic per launch of the kernel in an `ncu --set full` report.

    python tools/ncu_traffic.py REPORT WORKLOAD OUT_DIR [note]

Writes OUT_DIR/traffic_<WORKLOAD>.json = {kernel, dram_bytes_per_launch,
dram_read_bytes, dram_write_bytes, duration_ms, grid, note}; bench.py reports
it as roofline.traffic.
"""
import csv
import json
import os
import subprocess
import sys

_UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main():
    rep, workload, out_dir = sys.argv[1:4]
    note = sys.argv[4] if len(sys.argv) > 4 else ""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    head, units, vals = rows[0], rows[1], rows[2]

    def get(name):
        i = head.index(name)
        v = float(vals[i].replace(",", ""))
        return v * _UNITS.get(units[i], 1.0)

    rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
    i_t = head.index("gpu__time_duration.sum")
    dur = float(vals[i_t].replace(",", "")) * {"ms": 1.0, "us": 1e-3, "ns": 1e-6}.get(units[i_t], 1.0)
    res = {"kernel": vals[head.index("Kernel Name")], "dram_bytes_per_launch": rd + wr,
           "dram_read_bytes": rd, "dram_write_bytes": wr, "duration_ms": dur,
           "grid": vals[head.index("launch__grid_size")], "report": os.path.basename(rep),
           "note": note}
    os.makedirs(out_dir, exist_ok=True)
    path = os.path.join(out_dir, f"traffic_{workload}.json")
    with open(path, "w") as f:
        json.dump(res, f, indent=1)
    print(path, json.dumps(res))


if __name__ == "__main__":
    main()
