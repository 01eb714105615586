#!/usr/bin/env python
"""Summarise ncu captures into the JSON/markdown committed under profiles/ (developer tool, runs without a GPU).

    python tools/ncu_summary.py gpurun_out/<prof>.ncu-rep [...] > profiles/<name>.json
    python tools/ncu_summary.py --launches gpurun_out/<launches>.csv

For every kernel launch in a --set full capture: duration, SM clock, DRAM bytes read/written, DRAM throughput,
tensor-pipe and XU (MUFU) utilisation, registers, occupancy.  For a launch list (gpu__time_duration pass): the
per-kernel device times and each kernel's share of the step.
"""
from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict, defaultdict

METRICS = OrderedDict([
    ("gpu__time_duration.sum", "duration_ns"),
    ("sm__cycles_elapsed.avg.per_second", "sm_hz"),
    ("dram__bytes_read.sum", "dram_bytes_read"),
    ("dram__bytes_write.sum", "dram_bytes_write"),
    ("dram__bytes.sum.per_second", "dram_bytes_per_s"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct_of_peak"),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor_pipe_pct"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor_pipe_pct"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu_pipe_pct"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_throughput_pct"),
    ("launch__registers_per_thread", "registers"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved_occupancy_pct"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
])


def _num(s: str):
    s = s.replace(",", "").strip()
    try:
        return float(s)
    except ValueError:
        return s


def summarise_rep(path: str) -> list[dict]:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        rec = {"kernel": d.get("Kernel Name", "")[:120], "id": d.get("ID")}
        for m, key in METRICS.items():
            if m in d and d[m] != "":
                v = _num(d[m])
                u = units[hdr.index(m)]
                if isinstance(v, float) and u in ("Kbyte", "Mbyte", "Gbyte", "byte"):
                    v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
                if isinstance(v, float) and u in ("Kbyte/s", "Mbyte/s", "Gbyte/s", "Tbyte/s", "byte/s"):
                    v *= {"byte/s": 1, "Kbyte/s": 1e3, "Mbyte/s": 1e6, "Gbyte/s": 1e9, "Tbyte/s": 1e12}[u]
                if isinstance(v, float) and u in ("usecond", "msecond", "nsecond", "ns", "us", "ms", "s"):
                    v *= {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9}[u]
                if isinstance(v, float) and u in ("Ghz", "Mhz", "hz"):
                    v *= {"hz": 1, "Mhz": 1e6, "Ghz": 1e9}[u]
                rec[key] = v
        if "dram_bytes_read" in rec and "dram_bytes_write" in rec:
            rec["dram_bytes"] = rec["dram_bytes_read"] + rec["dram_bytes_write"]
        out.append(rec)
    return out


def summarise_launches(path: str) -> dict:
    rows = list(csv.reader(open(path)))
    hdr = None
    per = defaultdict(list)
    order = []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            name = d["Kernel Name"].split("(")[0]
            if name not in per:
                order.append(name)
            per[name].append(_num(d["Metric Value"]))
    return {name: {"launches": len(per[name]), "avg_ns": sum(per[name]) / len(per[name])} for name in order}


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        print(json.dumps(summarise_launches(sys.argv[2]), indent=1))
    else:
        print(json.dumps({p: summarise_rep(p) for p in sys.argv[1:]}, indent=1))
