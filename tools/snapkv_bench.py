#!/usr/bin/env python
"""SnapKV scorer microbenchmark (GPU): qvk_snapkv_score on the C3 shape (64 groups x 1024 tokens, 28 / 4 heads,
window 32) and C3b (64 x 4096), CUDA-event timed per launch after an L2 flush; one JSON line per shape.
QVK_BENCH_DRAIN=1: a ~100 us sleep kernel between the flush and the timed launch, so the flush's dirty L2 lines are
written back (and the launch is queued) before the first event — the kernel alone instead of kernel + write-back."""
import json
import os
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2505_16175_b200 as qp  # noqa: E402

dev = torch.device("cuda:0")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
drain = os.environ.get("QVK_BENCH_DRAIN") == "1"
for G, N in ((64, 1024), (64, 4096)):
    plan = qp.GroupPlan.from_sizes([N] * G, 0.25)
    g = plan.to(dev)
    q = torch.randn(G * N, 28, 128, device=dev).to(torch.bfloat16)
    k = torch.randn(G * N, 4, 128, device=dev).to(torch.bfloat16)
    sc = torch.empty(G * N * 4, dtype=torch.float64, device=dev)
    qp.snapkv_scores(q, k, g, 28, 4, 32, out=sc)
    ts = []
    for _ in range(20):
        flush.zero_()
        if drain:
            torch.cuda._sleep(200_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        qp.snapkv_scores(q, k, g, 28, 4, 32, out=sc)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    # the layer path: pass 1 comes out of the attention kernel (qvk_attention_window_stats), pass 2 alone here
    _, st = qp.attention_window_stats(q, k, k, g, 28, 4, 32)
    ts2 = []
    for _ in range(20):
        flush.zero_()
        if drain:
            torch.cuda._sleep(200_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        qp.snapkv_scores(q, k, g, 28, 4, 32, out=sc, window_stats=st)
        b.record()
        torch.cuda.synchronize()
        ts2.append(a.elapsed_time(b))
    ms2 = statistics.median(ts2)
    # the same launches back to back (as in the layer, where SnapKV follows the attention: no shared-memory carveout
    # switch, launch queued, K partly L2-resident) — what the isolated, flushed launches above add (~10 us at C3) is
    # launch / carveout / cold-cache cost
    ts3 = []
    for _ in range(5):
        torch.cuda.synchronize()
        torch.cuda._sleep(200_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            qp.snapkv_scores(q, k, g, 28, 4, 32, out=sc, window_stats=st)
        b.record()
        torch.cuda.synchronize()
        ts3.append(a.elapsed_time(b) / 20)
    ms3 = statistics.median(ts3)
    byt = G * N * 4 * 128 * 2 + G * 32 * 28 * 128 * 2 + G * N * 4 * 8
    exps = G * 4 * 7 * 32 * N  # exponentials of ONE pass (window rows x keys)
    floor_ms = 2 * exps / (16 * 148 * 1.965e9) * 1e3  # the MUFU floor of the two-exponential formulation
    print(json.dumps({"groups": G, "tokens": N, "ms": ms, "bytes": byt, "gbs": byt / ms / 1e6,
                      "mufu_floor_2exp_ms": floor_ms, "frac_of_mufu_floor": floor_ms / ms,
                      "pass2_ms": ms2, "mufu_floor_pass2_ms": floor_ms / 2, "pass2_frac_of_mufu_floor":
                      floor_ms / 2 / ms2, "pass2_back_to_back_ms": ms3,
                      "pass2_back_to_back_frac_of_mufu_floor": floor_ms / 2 / ms3}), flush=True)
