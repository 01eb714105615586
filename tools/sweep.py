#!/usr/bin/env python
"""Per-configuration measurements of the pruned-prefill path (BASELINE.json configs C1..C5), one JSON line each.

    python tools/sweep.py [--configs C1,C2,C3,C3b,C4,C5] [--steps 3] [--warmup 2] > profiles/rN_sweep.jsonl

bench.py keeps the driver contract on the headline config (C2); this tool covers the other rows of SURVEY.md §8(d):
  C1   tiny: 16 frames x 64 tok, group 4 frames, 4 Q / 2 KV heads, d 64, key-norm rho 0.5, 1 layer
  C2   7B layer: 256 frames x 256 tok, group 16, 28/4 heads, d 128, key-norm rho 0.5, 1 layer
  C3   7B SnapKV: 1024 frames x 64 tok (64 groups x 1024), SnapKV w=32 rho 0.25, 28 layers
  C3b  same with 256 tok/frame (64 groups x 4096)
  C4   1 h @ 1 FPS: 3600 frames x 256 tok (225 groups x 4096), key-norm rho 0.5, 28 layers (1 GPU holds all groups)
  C4L1 one C4 layer (225 groups x 4096) at rho {0.125, 0.25, 0.5}: the prune at the metric's scale
  C5   256 frames x 256 tok, group {4,8,16,32,64} frames x rho {0.125,0.25,0.5,1.0}, 1 layer
Per layer: one qvk_prefill_layer call (attention, then the prune: fused key-norm score+select+gather, or SnapKV
score + fused select+gather) into that layer's cache; a second, serialised pass times every kernel with CUDA events.  Layers use two alternating synthetic Q/K/V sets (each larger than L2, the
stand-in model has no residual stream: prefill.cpp:185-190), so timing is per-layer work on cold data.
tokens/s = tokens x layers-through / wall (a token counts once when it has gone through every layer).
"""
from __future__ import annotations

import argparse
import json
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
# the prune at the metric's scale (225 groups of 4096 tokens, ~12 waves of clusters) for every retention ratio
for rho in (0.125, 0.25, 0.5):
    CONFIGS[f"C4L1-r{rho}"] = dict(frames=3600, tpf=256, fpg=16, n_q=28, n_kv=4, d=128, layers=1,
                                   scorer="key_norm_small", rho=rho)
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
    win_stats = torch.empty(plan.n_groups, n_q, 32, dtype=torch.float32, device=dev) if snap else None
    scorer = qp.Scorer.snapkv if snap else qp.Scorer.key_norm_small
    times = {"attention": [], "score": [], "prune": []}

    def layer(l):
        """The production path: one qvk_prefill_layer call (attention, then the prune overlapping its tail)."""
        q, k, v = sets[l % len(sets)]
        buf = qp.LayerBuffers(o, scores, idx, kc[l], vc[l], org[l])
        qp.prefill_layer(q, k, v, g, n_q, n_kv, rho, scorer, True, buffers=buf)

    def layer_kernels(l):
        """Same layer with the kernels serialised and event-timed one by one (the roofline figures)."""
        q, k, v = sets[l % len(sets)]
        e = [ev() for _ in range(4)]
        e[0].record(stream)
        if snap and rho != 1.0:  # the production path: the attention also writes SnapKV's window statistics
            qp.attention_window_stats(q, k, v, g, n_q, n_kv, 32, out=o, stats=win_stats)
        else:
            qp.attention(q, k, v, g, n_q, n_kv, out=o)
        e[1].record(stream)
        if rho == 1.0:  # identity path: no scoring (prefill.cpp:263-270)
            e[2].record(stream)
            qp.gather(k, v, g, n_kv, d, None, kc[l], vc[l], org[l])
        elif snap:
            qp.snapkv_scores(q, k, g, n_q, n_kv, 32, 1, out=scores, window_stats=win_stats)
            e[2].record(stream)
            qp.select_gather(scores, k, v, g, n_kv, d, idx, kc[l], vc[l], org[l])
        else:
            e[2].record(stream)
            qp.lib.qvk_prune(stream.cuda_stream, g.ref, k.data_ptr(), v.data_ptr(), qp._lib.QVK_BF16, n_kv, d,
                             int(qp.Scorer.key_norm_small), rho, None, 0, n_kv, scores.data_ptr(), idx.data_ptr(),
                             kc[l].data_ptr(), vc[l].data_ptr(), org[l].data_ptr())
        e[3].record(stream)
        return e

    for _ in range(warmup):
        for l in range(L):
            layer(l)
    torch.cuda.synchronize()
    t0, t1 = ev(), ev()
    t0.record(stream)
    for _ in range(steps):
        for l in range(L):
            layer(l)
    t1.record(stream)
    torch.cuda.synchronize()
    wall_ms = t0.elapsed_time(t1)
    recs = [layer_kernels(l) for _ in range(max(1, steps // 2)) for l in range(min(L, 4))]
    torch.cuda.synchronize()
    for e in recs:
        times["attention"].append(e[0].elapsed_time(e[1]))
        times["score"].append(e[1].elapsed_time(e[2]))
        times["prune"].append(e[2].elapsed_time(e[3]))
    avg = {k_: statistics.mean(v_) for k_, v_ in times.items()}
    hbm, tf_burst, tf_sus, src = peaks()
    fl = flops_attention(sizes, n_q, d)
    T, Rr = plan.total_tokens, plan.total_rows
    if rho == 1.0:  # identity copy: K, V rows read and written, origin written
        b_prune = float(Rr * n_kv * (4 * d * 2 + 8))
        b_score = 0.0
    elif snap:  # snapkv.cu reads K and the window queries; the fused select/gather reads the scores
        b_score = snapkv_bytes(plan, n_q, n_kv, d, 32)
        b_prune = float(T * n_kv * 8 + Rr * n_kv * (4 * d * 2 + 8 + 4))
    else:  # fused prune (prune_fused.cu): K read once, scores written, retained V read, K/V/idx/origin written
        b_score = 0.0
        b_prune = bytes_prune(plan, n_kv, d)

    def gbs(b, ms):
        return None if ms <= 0 or b == 0 else b / (ms / 1e3) / 1e9

    out = {
        "config": name, **{k_: v_ for k_, v_ in c.items()}, "groups": plan.n_groups, "group_tokens": sizes[0],
        "tokens": T, "retained_rows": Rr, "steps": steps,
        "tokens_per_s": T * steps / (wall_ms / 1e3), "ms_per_step": wall_ms / steps,
        "path": "qvk_prefill_layer per layer (prune launched with PDL, overlapping the attention tail)",
        "attention": {"ms": avg["attention"], "tflops": fl / (avg["attention"] / 1e3) / 1e12,
                      "frac": fl / (avg["attention"] / 1e3) / 1e12 / tf_burst,
                      # the sustained peak (under the power cap) is the denominator for a kernel inside a long step
                      "frac_sustained": fl / (avg["attention"] / 1e3) / 1e12 / tf_sus if tf_sus else None},
        "prune": {"kernels": "identity gather" if rho == 1.0 else
                  ("snapkv score, then fused select+gather" if snap else "fused score+select+gather"),
                  "ms": avg["score"] + avg["prune"], "bytes": b_score + b_prune,
                  "gbs": gbs(b_score + b_prune, avg["score"] + avg["prune"]),
                  "frac": (gbs(b_score + b_prune, avg["score"] + avg["prune"]) or 0) / hbm},
        "peaks": {"tflops": tf_burst, "tflops_sustained": tf_sus, "hbm_gbs": hbm, "source": src},
    }
    if snap:
        # pass 2 only (pass 1 = the attention kernel's window statistics): one exponential per (window row of
        # each query head, key); its MUFU floor at 16 ex2 / clk / SM and the 1965 MHz boost clock
        exps = sum(int(n) * n_q * min(32, int(n)) for n in sizes)
        floor_ms = exps / (16 * 148 * 1.965e9) * 1e3
        out["snapkv_score"] = {"ms": avg["score"], "bytes": b_score, "gbs": gbs(b_score, avg["score"]),
                               "frac": (gbs(b_score, avg["score"]) or 0) / hbm,
                               "passes": "pass 2 only (window statistics from the attention kernel)",
                               "mufu_floor_ms": floor_ms, "frac_of_mufu_floor": floor_ms / avg["score"]}
        out["select_gather"] = {"ms": avg["prune"], "bytes": b_prune, "gbs": gbs(b_prune, avg["prune"]),
                                "frac": (gbs(b_prune, avg["prune"]) or 0) / hbm}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C3,C3b,C4,C4L1,C5")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    want = []
    for c in args.configs.split(","):
        want += [k for k in CONFIGS if k == c or (c in ("C5", "C4L1") and k.startswith(c + "-"))]
    for name in want:
        res = run(name, CONFIGS[name], args.steps, args.warmup, dev)
        print(json.dumps(res), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
