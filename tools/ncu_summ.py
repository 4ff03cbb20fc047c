#!/usr/bin/env python
"""Summarise ncu output for profiles/.

    python tools/ncu_summ.py report X.ncu-rep [--traffic-json out.json --tasks-per-launch T]
        one `--set full` report: key metrics per launch as markdown; optionally
        write the DRAM traffic per launch / per task (bench.py's roofline.traffic)
    python tools/ncu_summ.py launches X.csv
        a `--metrics gpu__time_duration.sum --csv` launch list: per-kernel count,
        share of the serialised time and mean duration as markdown

Reads reports with `ncu -i ... --page raw --csv` (ncu is in this image; no GPU needed).
"""
from __future__ import annotations

import collections
import csv
import io
import json
import re
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__cycles_elapsed.avg.per_second",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__cycles_active.avg", "sm__cycles_elapsed.avg",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "lts__t_sector_hit_rate.pct",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9,
         "second": 1}


def raw_rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    return hdr, units, data


def to_float(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return None


def report(path, traffic_json=None, tasks_per_launch=None):
    hdr, units, data = raw_rows(path)
    idx = {h: i for i, h in enumerate(hdr)}
    for r in data:
        print(f"### {r[idx['Kernel Name']][:90]}")
        print("| metric | value |\n|---|---|")
        for k in KEYS:
            if k in idx:
                print(f"| `{k}` | {r[idx[k]]} {units[idx[k]]} |")
        print()
    if traffic_json:
        r = data[0]
        rd = to_float(r[idx["dram__bytes_read.sum"]]) * SCALE.get(units[idx["dram__bytes_read.sum"]], 1)
        wr = to_float(r[idx["dram__bytes_write.sum"]]) * SCALE.get(units[idx["dram__bytes_write.sum"]], 1)
        t = (rd + wr)
        j = {"report": path, "kernel": r[idx["Kernel Name"]], "bytes_per_launch": t, "read": rd, "write": wr}
        if tasks_per_launch:
            j["tasks_per_launch"] = tasks_per_launch
            j["bytes_per_task"] = t / tasks_per_launch
        json.dump(j, open(traffic_json, "w"), indent=1)
        print(json.dumps(j))


def launches(path):
    txt = open(path).read()
    start = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[start:])))
    agg = collections.OrderedDict()
    total = 0.0
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r["Kernel Name"])[:60]
        unit = r["Metric Unit"]
        v = to_float(r["Metric Value"]) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}[unit]
        c, s = agg.get(name, (0, 0.0))
        agg[name] = (c + 1, s + v)
        total += v
    print(f"{sum(c for c, _ in agg.values())} launches, {total / 1e3:.1f} ms serialised\n")
    print("| kernel | launches | share | mean us |\n|---|---|---|---|")
    for name, (c, s) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{name}` | {c} | {s / total:.3f} | {s / c:.1f} |")


if __name__ == "__main__":
    if sys.argv[1] == "report":
        tj = sys.argv[sys.argv.index("--traffic-json") + 1] if "--traffic-json" in sys.argv else None
        tp = float(sys.argv[sys.argv.index("--tasks-per-launch") + 1]) if "--tasks-per-launch" in sys.argv else None
        report(sys.argv[2], tj, tp)
    else:
        launches(sys.argv[2])
