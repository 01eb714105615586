#!/usr/bin/env python
"""QKV projection microbenchmark (GPU): qvk_project_qkv (tcgen05 GEMM, with / without the fused key-norm) against
torch.matmul (cuBLAS) on the same bf16 operands, CUDA-event timed.  One JSON line per token count.

    python tools/project_bench.py [--reps 10]
    python tools/project_bench.py --sustained [--launches 20]   # C4 layer shape (921,600 tokens), launches back to
        back so the power cap engages; knobs (QVK_PROJ_WIDE, QVK_PROJ_2SM) are read once per process: A/B them
        with one process each
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2505_16175_b200 as qp  # noqa: E402


def timed(fn, reps):
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return statistics.median(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--sustained", action="store_true")
    ap.add_argument("--launches", type=int, default=20)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    d_model, n_q, n_kv, d_h = 3584, 28, 4, 128
    if args.sustained:
        T = 921600
        x = torch.randn(T, d_model, device=dev).to(torch.bfloat16)
        w = (torch.randn((n_q + 2 * n_kv) * d_h, d_model, device=dev) / d_model ** 0.5).to(torch.bfloat16)
        q = torch.empty(T, n_q, d_h, dtype=torch.bfloat16, device=dev)
        k = torch.empty(T, n_kv, d_h, dtype=torch.bfloat16, device=dev)
        v = torch.empty_like(k)
        fl = 2.0 * T * d_model * w.shape[0]
        r = {"tokens": T, "flop": fl, "launches": args.launches,
             "knobs": {kk: vv for kk, vv in __import__("os").environ.items() if kk.startswith("QVK_PROJ")}}
        ours = lambda: qp.project_qkv(x, w, n_q, n_kv, d_h, q=q, k=k, v=v)  # noqa: E731
        for name, f in (("ours", ours), ("cublas", lambda: torch.matmul(x, w.t()))):
            f()
            torch.cuda.synchronize()
            ts = []
            for _ in range(3):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(args.launches):
                    f()
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b) / args.launches)
            r[name] = {"ms": ts, "tflops": [fl / t / 1e9 for t in ts]}
            torch.cuda._sleep(500_000_000)  # ~0.25 s cool-down between the two
            torch.cuda.synchronize()
        print(json.dumps(r), flush=True)
        return
    for T in (16384, 65536):
        x = torch.randn(T, d_model, device=dev).to(torch.bfloat16)
        w = (torch.randn((n_q + 2 * n_kv) * d_h, d_model, device=dev) / d_model ** 0.5).to(torch.bfloat16)
        plan = qp.GroupPlan.from_sizes([4096] * (T // 4096), 0.5)
        g = plan.to(dev)
        q = torch.empty(T, n_q, d_h, dtype=torch.bfloat16, device=dev)
        k = torch.empty(T, n_kv, d_h, dtype=torch.bfloat16, device=dev)
        v = torch.empty_like(k)
        sc = torch.empty(T * n_kv, dtype=torch.float64, device=dev)
        out = torch.empty(T, w.shape[0], dtype=torch.bfloat16, device=dev)
        ours = lambda: qp.project_qkv(x, w, n_q, n_kv, d_h, q=q, k=k, v=v)  # noqa: E731
        fused = lambda: qp.project_qkv(x, w, n_q, n_kv, d_h, g, True, q, k, v, sc)  # noqa: E731
        cublas = lambda: torch.matmul(x, w.t(), out=out)  # noqa: E731
        for f in (ours, fused, cublas):
            f()
        torch.cuda.synchronize()
        fl = 2.0 * T * d_model * w.shape[0]
        r = {"tokens": T, "flop": fl}
        for name, f in (("ours", ours), ("ours_fused_keynorm", fused), ("cublas", cublas)):
            ms = timed(f, args.reps)
            r[name] = {"ms": ms, "tflops": fl / ms / 1e9}
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
