#!/usr/bin/env python
"""Summarise an ncu report (.ncu-rep) into JSON: per-kernel duration, DRAM bytes, throughputs.

    python tools/ncu_summary.py gpurun_out/prof_matvec_r01.ncu-rep [--cells N] > profiles/...json
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes.sum.per_second",
        "lts__t_bytes.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9, "s": 1.0}


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                v = r[i].replace(",", "")
                try:
                    x = float(v)
                except ValueError:
                    continue
                u = units[i]
                if u in SCALE:
                    x *= SCALE[u]
                    u = "s" if u.endswith("s") or u.endswith("second") else "byte"
                elif u.endswith("/s") and u.split("/")[0] in SCALE:
                    x *= SCALE[u.split("/")[0]]
                    u = "byte/s"
                d[k] = x
                d[k + ".unit"] = u
        res.append(d)
    return res


if __name__ == "__main__":
    path = sys.argv[1]
    cells = None
    if "--cells" in sys.argv:
        cells = float(sys.argv[sys.argv.index("--cells") + 1])
    ks = load(path)
    for d in ks:
        d["dram_bytes_per_launch"] = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        if cells:
            d["dram_bytes_per_cell"] = d["dram_bytes_per_launch"] / cells
    json.dump({"source": path, "kernels": ks}, sys.stdout, indent=1)
    print()
