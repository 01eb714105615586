#!/usr/bin/env python
"""Copy one gpu_session.sh session's results into profiles/ (developer tool, runs without a GPU):

    python tools/update_profiles.py gpurun_out/<tag> [--round r2]

bench line / reference-arm line -> profiles/<round>_bench_line.json / _bench_reference_line.json; the ncu --set full
captures of the bench's attention and fused prune -> profiles/ncu_attention_c4_summary.json /
ncu_prune_c4_summary.json (bench.py reads `dram_bytes_per_launch` from them as roofline.traffic); the SnapKV
captures -> profiles/<round>_ncu_snapkv_c3.json; the launch list -> profiles/<round>_launches.{csv,json}; the sweep
-> profiles/<round>_sweep.jsonl.  Files a session did not produce are left alone.
"""
from __future__ import annotations

import argparse
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
PROF = ROOT / "profiles"


def last_json_line(path: Path):
    lines = [x for x in path.read_text().splitlines() if x.startswith("{")]
    return json.loads(lines[-1]) if lines else None


def ncu_summary(rep: Path):
    out = subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_summary.py"), str(rep)], capture_output=True,
                         text=True, check=True).stdout
    return list(json.loads(out).values())[0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("session")
    ap.add_argument("--round", default="r2")
    a = ap.parse_args()
    ses = Path(a.session)
    tag = ses.name
    for src, dst in (("bench.log", f"{a.round}_bench_line.json"), ("bench_ref.log", f"{a.round}_bench_reference_line.json")):
        if (ses / src).exists() and (d := last_json_line(ses / src)):
            (PROF / dst).write_text(json.dumps(d, indent=1))
            print("wrote", dst)
    if (ses / "attn.ncu-rep").exists():
        k = ncu_summary(ses / "attn.ncu-rep")[0]
        (PROF / "ncu_attention_c4_summary.json").write_text(json.dumps({
            "kernel": k["kernel"], "dram_bytes_per_launch": k["dram_bytes"], "dram_bytes_read": k["dram_bytes_read"],
            "dram_bytes_write": k["dram_bytes_write"], "algorithmic_bytes": 15099494400,
            "duration_ns_under_ncu": k["duration_ns"], "sm_hz_under_ncu": k["sm_hz"],
            "tensor_pipe_pct": k["tensor_pipe_pct"], "xu_pipe_pct": k["xu_pipe_pct"], "registers": k["registers"],
            "source": f"ncu --set full --clock-control none --import-source on (gpurun_out/{tag}/attn.ncu-rep), "
                      "bench.py C4 (225 groups x 4096 tokens, one layer per launch), third launch"}, indent=1))
        print("wrote ncu_attention_c4_summary.json")
    if (ses / "prune.ncu-rep").exists():
        k = ncu_summary(ses / "prune.ncu-rep")[0]
        (PROF / "ncu_prune_c4_summary.json").write_text(json.dumps({
            "kernel": k["kernel"], "dram_bytes_per_launch": k["dram_bytes"], "dram_bytes_read": k["dram_bytes_read"],
            "dram_bytes_write": k["dram_bytes_write"], "algorithmic_bytes": 2410905600.0,
            "duration_ns_under_ncu": k["duration_ns"], "sm_hz_under_ncu": k["sm_hz"],
            "dram_pct_of_peak": k["dram_pct_of_peak"], "registers": k["registers"],
            "achieved_occupancy_pct": k["achieved_occupancy_pct"], "grid": k["grid"],
            "source": f"ncu --set full --clock-control none --import-source on (gpurun_out/{tag}/prune.ncu-rep), "
                      "bench.py C4, third launch"}, indent=1))
        print("wrote ncu_prune_c4_summary.json")
    snap = {}
    for nm, what in (("snap", "two-pass qvk_snapkv_score, C3 (64 groups x 1024 tokens, 28/4 heads, window 32)"),
                     ("snap2", "pass 2 only (qvk_snapkv_score_stats on the attention kernel's window statistics), C3")):
        if (ses / f"{nm}.ncu-rep").exists():
            k = ncu_summary(ses / f"{nm}.ncu-rep")[0]
            k["what"] = what
            snap[nm] = k
    if snap:
        snap["source"] = f"ncu --set full --clock-control none (gpurun_out/{tag}/snap*.ncu-rep), tools/snapkv_bench.py"
        (PROF / f"{a.round}_ncu_snapkv_c3.json").write_text(json.dumps(snap, indent=1))
        print(f"wrote {a.round}_ncu_snapkv_c3.json")
    if (ses / "launches.csv").exists():
        shutil.copy(ses / "launches.csv", PROF / f"{a.round}_launches.csv")
        out = subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_summary.py"), "--launches",
                              str(ses / "launches.csv")], capture_output=True, text=True, check=True).stdout
        (PROF / f"{a.round}_launches.json").write_text(out)
        print(f"wrote {a.round}_launches.*")
    if (ses / "sweep.jsonl").exists() and (ses / "sweep.jsonl").stat().st_size > 0:
        shutil.copy(ses / "sweep.jsonl", PROF / f"{a.round}_sweep.jsonl")
        print(f"wrote {a.round}_sweep.jsonl")


if __name__ == "__main__":
    main()
