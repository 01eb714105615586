#!/usr/bin/env python
"""CTA-pair attention (attention2.cu, QVK_ATTN_2CTA=1) vs the one-CTA kernel: correctness against torch fp32 on ragged
shapes, then event-timed throughput of both on C2 / C3 / C4-layer shapes.  One JSON line per item."""
import json
import math
import os
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import torch  # noqa: E402

import paper_2505_16175_b200 as qp  # noqa: E402
from test_kernels_gpu import torch_attention  # noqa: E402

dev = torch.device("cuda", 0)


def run(q, k, v, g, n_q, n_kv, two):
    os.environ["QVK_ATTN_2CTA"] = "1" if two else "0"
    return qp.attention(q, k, v, g, n_q, n_kv)


def mk(sizes, n_q, n_kv, seed=1):
    q = torch.cat([qp.synth_bf16(seed, 3, 0, i, n, n_q, 128, False, dev) for i, n in enumerate(sizes)])
    k = torch.cat([qp.synth_bf16(seed, 1, 0, i, n, n_kv, 128, True, dev) for i, n in enumerate(sizes)])
    v = torch.cat([qp.synth_bf16(seed, 2, 0, i, n, n_kv, 128, False, dev) for i, n in enumerate(sizes)])
    return q, k, v


for sizes, n_q, n_kv in (([256], 2, 1), ([128], 1, 1), ([384, 100, 1, 129], 28, 4), ([4096], 28, 4),
                         ([1000, 37, 4096], 28, 4), ([255, 257, 513], 8, 2)):
    q, k, v = mk(sizes, n_q, n_kv)
    g = qp.GroupPlan.from_sizes(sizes, 0.5).to(dev)
    o2 = run(q, k, v, g, n_q, n_kv, True)
    o1 = run(q, k, v, g, n_q, n_kv, False)
    torch.cuda.synchronize()
    ref = torch_attention(q, k, v, sizes, n_q, n_kv, 1 / math.sqrt(128))
    err = (o2.float() - ref).abs()
    bad = (err > 1e-2 + 1e-2 * ref.abs()).sum().item()
    print(json.dumps({"item": "check", "sizes": sizes, "n_q": n_q, "bad": bad, "max_err": err.max().item(),
                      "max_err_1cta": (o1.float() - ref).abs().max().item()}), flush=True)

for name, G, N in (("C2", 16, 4096), ("C3", 64, 1024), ("C4_layer", 225, 4096)):
    sizes = [N] * G
    q, k, v = mk(sizes, 28, 4)
    g = qp.GroupPlan.from_sizes(sizes, 0.5).to(dev)
    fl = sum(4.0 * 128 * 28 * n * (n + 1) / 2 for n in sizes)
    for two in (False, True, False, True):
        for _ in range(2):
            run(q, k, v, g, 28, 4, two)
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            run(q, k, v, g, 28, 4, two)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = statistics.median(ts)
        print(json.dumps({"item": "perf", "config": name, "variant": "2cta" if two else "1cta", "ms": ms,
                          "tflops": fl / ms / 1e9}), flush=True)
    del q, k, v
    torch.cuda.empty_cache()
