#!/usr/bin/env python
"""Decode-consumer microbenchmark (GPU): qvk_decode_attention over a pruned cache, CUDA-event timed after a 256 MB
L2 flush.  Algorithmic bytes = K + V cache read once (2 * rows * n_kv * d * 2) + q + o; one JSON line per case.

    python tools/decode_bench.py [--reps 20]
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2505_16175_b200 as qp  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    n_q, n_kv, d = 28, 4, 128
    for name, rows in (("C2 cache (16 x 2048 rows)", 32768), ("C4 layer cache (225 x 2048 rows)", 460800)):
        kc = torch.randn(rows, n_kv, d, device=dev).to(torch.bfloat16)
        vc = torch.randn(rows, n_kv, d, device=dev).to(torch.bfloat16)
        for n_tq in (1, 16, 64):
            q = torch.randn(n_tq, n_q, d, device=dev).to(torch.bfloat16)
            o = torch.empty_like(q)
            qp.decode_attention(q, kc, vc, n_q, n_kv, out=o)
            ts = []
            for _ in range(args.reps):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                qp.decode_attention(q, kc, vc, n_q, n_kv, out=o)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            ms = statistics.median(ts)
            byt = 2 * rows * n_kv * d * 2 + 2 * q.numel() * 2
            fl = 4.0 * n_tq * n_q * rows * d
            print(json.dumps({"cache": name, "rows": rows, "query_tokens": n_tq, "ms": ms, "bytes": byt,
                              "gbs": byt / ms / 1e6, "hbm_frac": byt / ms / 1e6 / 6650.0,
                              "tflops": fl / ms / 1e9}), flush=True)


if __name__ == "__main__":
    main()
