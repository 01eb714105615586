#!/usr/bin/env python
"""One pruned-prefill layer with the SnapKV scorer (qvk_prefill_layer: attention -> SnapKV score -> select + gather)
on the C3 / C3b group shapes, CUDA-event timed after an L2 flush; one JSON line per shape.  Run with
QVK_SNAPKV_LSE=0 to time the two-pass scorer (its own pass 1) instead of the attention's window statistics."""
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
for G, N in ((64, 1024), (64, 4096)):
    plan = qp.GroupPlan.from_sizes([N] * G, 0.25)
    g = plan.to(dev)
    q = torch.randn(G * N, 28, 128, device=dev).to(torch.bfloat16)
    k = torch.randn(G * N, 4, 128, device=dev).to(torch.bfloat16)
    v = torch.randn(G * N, 4, 128, device=dev).to(torch.bfloat16)
    buf = qp.prefill_layer(q, k, v, g, 28, 4, 0.25, qp.Scorer.snapkv, True)
    res = {}
    for what in ("layer", "attention"):
        ts = []
        for _ in range(15):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            if what == "layer":
                qp.prefill_layer(q, k, v, g, 28, 4, 0.25, qp.Scorer.snapkv, True, buffers=buf)
            else:
                qp.attention(q, k, v, g, 28, 4, out=buf.o)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        res[what] = statistics.median(ts)
    print(json.dumps({"groups": G, "tokens": N, "lse": os.environ.get("QVK_SNAPKV_LSE", "1"),
                      "layer_ms": res["layer"], "attention_ms": res["attention"],
                      "prune_ms": res["layer"] - res["attention"]}), flush=True)
