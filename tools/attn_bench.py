#!/usr/bin/env python
"""Attention microbenchmark (GPU): qvk_attention on the BASELINE group shapes (inputs larger than L2), median of
--reps, one JSON line per shape.  A/B: QVK_LIB_PATH=build/ab/<rev>/libqvk.so.
  --mode burst (default): isolated launches — each queued behind a ~50 us sleep kernel, so the host's launch latency
     (~20-50 us of ctypes + tensor-map encoding, 4-10 % of a 0.5 ms C3 launch) is not on the device clock, with a
     pause between repetitions so the clocks stay at boost (the burst peak's conditions);
  --mode sustained: --batch back-to-back launches per measurement after ~1 s of warm-up (the power cap engages).

    python tools/attn_bench.py [--reps 20]
"""
import argparse
import json
import math
import statistics
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2505_16175_b200 as qp  # noqa: E402

SHAPES = [("C2", 16, 4096), ("C3", 64, 1024), ("C3-long", 16, 1024), ("C5-g8", 32, 2048), ("C5-g64", 4, 16384)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--batch", type=int, default=10)
    ap.add_argument("--mode", choices=["burst", "sustained"], default="burst")
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
        if args.mode == "burst":
            for _ in range(3):
                qp.attention(q, k, v, g, n_q, n_kv, 1 / math.sqrt(d), out=o)
            ts = []
            for _ in range(args.reps):
                torch.cuda.synchronize()
                time.sleep(0.05)
                torch.cuda._sleep(100_000)  # ~50 us: the launch below is queued before the first event fires
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                qp.attention(q, k, v, g, n_q, n_kv, 1 / math.sqrt(d), out=o)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            ms = statistics.median(ts)
            fl = 4.0 * d * n_q * N * (N + 1) / 2 * G
            print(json.dumps({"shape": name, "mode": "burst", "groups": G, "group_tokens": N, "ms": ms,
                              "tflops": fl / ms / 1e9}), flush=True)
            del q, k, v, o
            continue
        w0 = torch.cuda.Event(enable_timing=True)
        w0.record()
        while True:  # warm-up: ~1 s of launches
            for _ in range(args.batch):
                qp.attention(q, k, v, g, n_q, n_kv, 1 / math.sqrt(d), out=o)
            w1 = torch.cuda.Event(enable_timing=True)
            w1.record()
            torch.cuda.synchronize()
            if w0.elapsed_time(w1) > 1000.0:
                break
        ts = []
        for _ in range(args.reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(args.batch):
                qp.attention(q, k, v, g, n_q, n_kv, 1 / math.sqrt(d), out=o)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) / args.batch)
        ms = statistics.median(ts)
        fl = 4.0 * d * n_q * N * (N + 1) / 2 * G
        print(json.dumps({"shape": name, "mode": "sustained", "groups": G, "group_tokens": N, "ms": ms,
                          "tflops": fl / ms / 1e9}), flush=True)
        del q, k, v, o


if __name__ == "__main__":
    main()
