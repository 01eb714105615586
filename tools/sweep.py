#!/usr/bin/env python
"""Per-configuration measurements of the pruned-prefill path (BASELINE.json configs C1..C5), one JSON line each.

    python tools/sweep.py [--configs C1,C2,C3,C3b,C4,C5] [--steps 3] [--warmup 2] > profiles/rN_sweep.jsonl

bench.py keeps the driver contract on the headline config (C2); this tool covers the other rows of SURVEY.md §8(d):
  C1   tiny: 16 frames x 64 tok, group 4 frames, 4 Q / 2 KV heads, d 64, key-norm rho 0.5, 1 layer
  C2   7B layer: 256 frames x 256 tok, group 16, 28/4 heads, d 128, key-norm rho 0.5, 1 layer
  C3   7B SnapKV: 1024 frames x 64 tok (64 groups x 1024), SnapKV w=32 rho 0.25, 28 layers
  C3b  same with 256 tok/frame (64 groups x 4096)
  C4   1 h @ 1 FPS: 3600 frames x 256 tok (225 groups x 4096), key-norm rho 0.5, 28 layers (1 GPU holds all groups)
  C5   256 frames x 256 tok, group {4,8,16,32,64} frames x rho {0.125,0.25,0.5,1.0}, 1 layer
Per layer: attention -> score (key-norm or SnapKV) -> select -> gather into that layer's cache, every kernel timed
with CUDA events on the launch stream.  Layers use two alternating synthetic Q/K/V sets (each larger than L2, the
stand-in model has no residual stream: prefill.cpp:185-190), so timing is per-layer work on cold data.
tokens/s = tokens x layers-through / wall (a token counts once when it has gone through every layer).
"""
from __future__ import annotations

import argparse
import json
import math
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2505_16175_b200 as qp  # noqa: E402
from bench import bytes_prune, flops_attention, peaks  # noqa: E402

CONFIGS = {
    "C1": dict(frames=16, tpf=64, fpg=4, n_q=4, n_kv=2, d=64, layers=1, scorer="key_norm_small", rho=0.5),
    "C2": dict(frames=256, tpf=256, fpg=16, n_q=28, n_kv=4, d=128, layers=1, scorer="key_norm_small", rho=0.5),
    "C3": dict(frames=1024, tpf=64, fpg=16, n_q=28, n_kv=4, d=128, layers=28, scorer="snapkv", rho=0.25),
    "C3b": dict(frames=1024, tpf=256, fpg=16, n_q=28, n_kv=4, d=128, layers=28, scorer="snapkv", rho=0.25),
    "C4": dict(frames=3600, tpf=256, fpg=16, n_q=28, n_kv=4, d=128, layers=28, scorer="key_norm_small", rho=0.5),
}
for fpg in (4, 8, 16, 32, 64):
    for rho in (0.125, 0.25, 0.5, 1.0):
        CONFIGS[f"C5-g{fpg}-r{rho}"] = dict(frames=256, tpf=256, fpg=fpg, n_q=28, n_kv=4, d=128, layers=1,
                                            scorer="key_norm_small", rho=rho)


def snapkv_bytes(plan, n_q, n_kv, d, w):
    T = plan.total_tokens
    win = sum(min(w, int(n)) for n in plan.sizes)
    return float(T * n_kv * d * 2 + win * n_q * d * 2 + T * n_kv * 8)


def run(name, c, steps, warmup, dev):
    n_q, n_kv, d, L, rho = c["n_q"], c["n_kv"], c["d"], c["layers"], c["rho"]
    plan = qp.GroupPlan.plan(c["frames"], c["fpg"], c["tpf"], rho, 1)
    g = plan.to(dev)
    sizes = [int(s) for s in plan.sizes]
    sets = []
    for s_ in range(2 if L > 1 else 1):
        sets.append(tuple(torch.cat([qp.synth_bf16(1 + s_, tag, 0, i, n, h, d, tag == 1, dev)
                                     for i, n in enumerate(sizes)]) for tag, h in ((3, n_q), (1, n_kv), (2, n_kv))))
    R = plan.total_rows
    kc = torch.empty(L, R * n_kv * d, dtype=torch.bfloat16, device=dev)
    vc = torch.empty_like(kc)
    org = torch.empty(L, R * n_kv, dtype=torch.int64, device=dev)
    o = torch.empty_like(sets[0][0])
    scores = torch.empty(plan.total_tokens * n_kv, dtype=torch.float64, device=dev)
    idx = torch.empty(max(1, R * n_kv), dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    snap = c["scorer"] == "snapkv"
    times = {"attention": [], "score": [], "select": [], "gather": []}

    def layer(l, rec):
        q, k, v = sets[l % len(sets)]
        e = [ev() for _ in range(5)]
        e[0].record(stream)
        qp.attention(q, k, v, g, n_q, n_kv, out=o)
        e[1].record(stream)
        if rho != 1.0:
            if snap:
                qp.snapkv_scores(q, k, g, n_q, n_kv, 32, 1, out=scores)
            else:
                qp.score(k, v, g, n_kv, d, qp.Scorer.key_norm_small, out=scores)
            e[2].record(stream)
            qp.select(scores, g, n_kv, out=idx)
            e[3].record(stream)
            qp.gather(k, v, g, n_kv, d, idx, kc[l], vc[l], org[l])
        else:  # identity path: no scoring (prefill.cpp:263-270)
            e[2].record(stream)
            e[3].record(stream)
            qp.gather(k, v, g, n_kv, d, None, kc[l], vc[l], org[l])
        e[4].record(stream)
        if rec is not None:
            rec.append(e)

    for _ in range(warmup):
        for l in range(L):
            layer(l, None)
    torch.cuda.synchronize()
    t0, t1 = ev(), ev()
    recs = []
    t0.record(stream)
    for _ in range(steps):
        for l in range(L):
            layer(l, recs)
    t1.record(stream)
    torch.cuda.synchronize()
    wall_ms = t0.elapsed_time(t1)
    for e in recs:
        times["attention"].append(e[0].elapsed_time(e[1]))
        times["score"].append(e[1].elapsed_time(e[2]))
        times["select"].append(e[2].elapsed_time(e[3]))
        times["gather"].append(e[3].elapsed_time(e[4]))
    avg = {k_: statistics.mean(v_) for k_, v_ in times.items()}
    hbm, tf_burst, _, src = peaks()
    fl = flops_attention(sizes, n_q, d)
    T, Rr = plan.total_tokens, plan.total_rows
    b_score = snapkv_bytes(plan, n_q, n_kv, d, 32) if snap else float(T * n_kv * (d * 2 + 8))
    b_select = float(T * n_kv * 8 + Rr * n_kv * 4)
    b_gather = float(Rr * n_kv * (4 * d * 2 + 8 + (4 if rho != 1.0 else 0)))
    if rho == 1.0:
        b_score = b_select = 0.0

    def gbs(b, ms):
        return None if ms <= 0 or b == 0 else b / (ms / 1e3) / 1e9

    out = {
        "config": name, **{k_: v_ for k_, v_ in c.items()}, "groups": plan.n_groups, "group_tokens": sizes[0],
        "tokens": T, "retained_rows": Rr, "steps": steps,
        "tokens_per_s": T * steps / (wall_ms / 1e3), "ms_per_step": wall_ms / steps,
        "attention": {"ms": avg["attention"], "tflops": fl / (avg["attention"] / 1e3) / 1e12,
                      "frac": fl / (avg["attention"] / 1e3) / 1e12 / tf_burst},
        "score": {"kernel": "snapkv" if snap else "key_norm", "ms": avg["score"], "bytes": b_score,
                  "gbs": gbs(b_score, avg["score"]),
                  "frac": (gbs(b_score, avg["score"]) or 0) / hbm},
        "select": {"ms": avg["select"], "bytes": b_select, "gbs": gbs(b_select, avg["select"])},
        "gather": {"ms": avg["gather"], "bytes": b_gather, "gbs": gbs(b_gather, avg["gather"]),
                   "frac": (gbs(b_gather, avg["gather"]) or 0) / hbm},
        "prune": {"ms": avg["score"] + avg["select"] + avg["gather"],
                  "frac": ((b_score + b_select + b_gather) /
                           max(1e-9, (avg["score"] + avg["select"] + avg["gather"]) / 1e3) / 1e9) / hbm},
        "peaks": {"tflops": tf_burst, "hbm_gbs": hbm, "source": src},
    }
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C3,C3b,C4,C5")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    want = []
    for c in args.configs.split(","):
        want += [k for k in CONFIGS if k == c or (c == "C5" and k.startswith("C5-"))]
    for name in want:
        res = run(name, CONFIGS[name], args.steps, args.warmup, dev)
        print(json.dumps(res), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
