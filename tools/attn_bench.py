#!/usr/bin/env python
"""Attention microbenchmark (GPU): qvk_attention on the BASELINE group shapes, CUDA-event timed per launch (median of
--reps after warm-up; inputs larger than L2).  One JSON line per shape.  A/B: QVK_LIB_PATH=build/ab/<rev>/libqvk.so.

    python tools/attn_bench.py [--reps 20]
"""
import argparse
import json
import math
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2505_16175_b200 as qp  # noqa: E402

SHAPES = [("C2", 16, 4096), ("C3", 64, 1024), ("C3-long", 16, 1024), ("C5-g8", 32, 2048), ("C5-g64", 4, 16384)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    n_q, n_kv, d = 28, 4, 128
    for name, G, N in SHAPES:
        sizes = [N] * G
        plan = qp.GroupPlan.from_sizes(sizes, 0.5)
        g = plan.to(dev)
        T = G * N
        q = torch.randn(T, n_q, d, device=dev).to(torch.bfloat16)
        k = torch.randn(T, n_kv, d, device=dev).to(torch.bfloat16)
        v = torch.randn(T, n_kv, d, device=dev).to(torch.bfloat16)
        o = torch.empty_like(q)
        for _ in range(3):
            qp.attention(q, k, v, g, n_q, n_kv, 1 / math.sqrt(d), out=o)
        ts = []
        for _ in range(args.reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            qp.attention(q, k, v, g, n_q, n_kv, 1 / math.sqrt(d), out=o)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = statistics.median(ts)
        fl = 4.0 * d * n_q * N * (N + 1) / 2 * G
        print(json.dumps({"shape": name, "groups": G, "group_tokens": N, "ms": ms, "tflops": fl / ms / 1e9}), flush=True)
        del q, k, v, o


if __name__ == "__main__":
    main()
