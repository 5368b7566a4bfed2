#!/usr/bin/env python
"""Summarise ncu output for profiles/: launch-list shares and the key counters of a --set full capture.

  python scripts/ncu_summary.py launches <launches.csv>            -> per-kernel time share (json)
  python scripts/ncu_summary.py full <prof.ncu-rep> [kernel-regex]   -> key metrics per profiled launch (json)
"""
import csv
import io
import json
import re
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ix = {h: i for i, h in enumerate(hdr)}
    agg = {}
    for r in rows[start + 1:]:
        if len(r) < len(hdr) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r[ix["Kernel Name"]]).split("::")[-1]
        v = float(r[ix["Metric Value"]].replace(",", ""))
        unit = r[ix["Metric Unit"]]
        ns = v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ns
    tot = sum(v[1] for v in agg.values())
    return {k: {"launches": v[0], "total_ms": v[1] / 1e6, "avg_ms": v[1] / v[0] / 1e6, "share": v[1] / tot}
            for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])}


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed.sum", "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
        "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct", "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def full(path, kregex=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    units = rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", "")
        if kregex and not re.search(kregex, name):
            continue
        m = {"kernel": re.sub(r"\(.*", "", name)}
        for k in KEYS:
            if k in d:
                u = units[hdr.index(k)]
                m[k] = d[k] + (f" {u}" if u else "")
        res.append(m)
    return res


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        print(json.dumps(launches(sys.argv[2]), indent=1))
    else:
        print(json.dumps(full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None), indent=1))
