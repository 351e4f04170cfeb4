"""Summarise ncu outputs into profiles/ (launch list CSV + one --set full report)."""
import csv
import json
import subprocess
import sys
from collections import defaultdict


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hdr]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    per = defaultdict(lambda: defaultdict(list))
    ids = {}
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        per[name][r[mi]].append(float(r[vi].replace(",", "")))
    out = {}
    tot = sum(sum(m.get("gpu__time_duration.sum", [])) for m in per.values())
    for k, m in per.items():
        t = m.get("gpu__time_duration.sum", [])
        out[k] = {"launches": len(t), "avg_us": round(sum(t) / len(t) / 1e3, 2) if t else None,
                  "share_of_time": round(sum(t) / tot, 4) if tot else None}
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            if m.get(key):
                out[k][key + "_avg"] = sum(m[key]) / len(m[key])
    return out


def full(rep, names):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    out = {}
    for i, n in enumerate(h):
        if n in names or n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("per_issue_active.ratio"):
            out[n] = v[i] + (" " + u[i] if u[i] else "")
    return out


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "launches":
        print(json.dumps(launches(sys.argv[2]), indent=1))
    else:
        keys = {"gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
                "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
                "launch__grid_size", "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum",
                "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed"}
        print(json.dumps(full(sys.argv[2], keys), indent=1))
