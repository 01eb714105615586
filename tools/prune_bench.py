#!/usr/bin/env python
"""Prune-path microbenchmark (GPU): the fused one-launch kernel (qvk_prune -> prune_fused.cu) against the three
separate launches (qvk_score, qvk_select, qvk_gather), CUDA-event timed per launch with an L2 flush (256 MB write)
between repetitions.  Prints one JSON line per configuration.

    python tools/prune_bench.py [--reps 20]
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2505_16175_b200 as qp  # noqa: E402


def timed(fn, reps, flush):
    out = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return statistics.median(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--only", default=None, help="run one configuration (e.g. C2)")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    hbm = 6650.0
    cfgs = [("C2", 16, 4096, 4, 128, 0.5), ("C4-layer", 225, 4096, 4, 128, 0.5), ("C3", 64, 1024, 4, 128, 0.25),
            ("C5-g64", 4, 16384, 4, 128, 0.125), ("C1", 4, 256, 2, 64, 0.5), ("per-token", 16, 4096, 1, 512, 0.5),
            ("per-token-256", 16, 4096, 1, 256, 0.5), ("per-token-C4", 225, 4096, 1, 512, 0.5)]
    for name, G, N, H, D, rho in cfgs:
        if args.only and name != args.only:
            continue
        sizes = [N] * G
        plan = qp.GroupPlan.from_sizes(sizes, rho)
        g = plan.to(dev)
        k = torch.cat([qp.synth_bf16(1, 1, 0, i, N, H, D, True, dev) for i in range(G)])
        v = torch.cat([qp.synth_bf16(1, 2, 0, i, N, H, D, False, dev) for i in range(G)])
        T, R = plan.total_tokens, plan.total_rows
        sc = torch.empty(T * H, dtype=torch.float64, device=dev)
        ix = torch.empty(R * H, dtype=torch.int32, device=dev)
        kc = torch.empty(R * H * D, dtype=torch.bfloat16, device=dev)
        vc = torch.empty_like(kc)
        og = torch.empty(R * H, dtype=torch.int64, device=dev)
        s = torch.cuda.current_stream().cuda_stream
        ks = int(qp.Scorer.key_norm_small)

        def fused():
            qp.lib.qvk_prune(s, g.ref, k.data_ptr(), v.data_ptr(), qp._lib.QVK_BF16, H, D, ks, rho, None, 0, H,
                             sc.data_ptr(), ix.data_ptr(), kc.data_ptr(), vc.data_ptr(), og.data_ptr())

        def separate():
            qp.score(k, v, g, H, D, qp.Scorer.key_norm_small, out=sc)
            qp.select(sc, g, H, out=ix)
            qp.gather(k, v, g, H, D, ix, kc, vc, og)

        def score_only():
            qp.score(k, v, g, H, D, qp.Scorer.key_norm_small, out=sc)

        def sg_only():
            qp.select_gather(sc, k, v, g, H, D, ix, kc, vc, og)

        def two_kernels():
            score_only()
            sg_only()

        for f in (fused, separate, two_kernels):
            f()
        torch.cuda.synchronize()
        tf, ts = timed(fused, args.reps, flush), timed(separate, args.reps, flush)
        t2, t_sc, t_sg = (timed(f, args.reps, flush) for f in (two_kernels, score_only, sg_only))
        alg = T * H * (2 * D + 8) + R * H * (6 * D + 12)
        print(json.dumps({"config": name, "G": G, "N": N, "heads": H, "width": D, "rho": rho,
                          "fused_us": tf * 1e3, "separate_us": ts * 1e3, "alg_bytes": alg,
                          "fused_gbs": alg / tf / 1e6, "fused_frac_hbm": alg / tf / 1e6 / hbm,
                          "separate_gbs": alg / ts / 1e6, "score_then_select_gather_us": t2 * 1e3,
                          "score_us": t_sc * 1e3, "select_gather_us": t_sg * 1e3}), flush=True)


if __name__ == "__main__":
    main()
