#!/usr/bin/env python
"""Where a C4 step's time goes between the layers (developer tool): 8 consecutive C4 layers (225 groups x 4096
tokens, 28 / 4 heads) timed with CUDA events as (A) qvk_prefill_layer (attention + fused prune with PDL), (B) the
attention alone, (C) attention then a standalone qvk_prune; ms per layer for each, repeated."""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2505_16175_b200 as qp  # noqa: E402

dev = torch.device("cuda:0")
G, N, NQ, NKV, D, L = 225, 4096, 28, 4, 128, 8
plan = qp.GroupPlan.from_sizes([N] * G, 0.5)
g = plan.to(dev)
sets = [tuple(torch.cat([qp.synth_bf16(1, tag, s_, i, N, h, D, tag == 1, dev) for i in range(G)])
              for tag, h in ((3, NQ), (1, NKV), (2, NKV))) for s_ in range(2)]
buf = qp.LayerBuffers.allocate(plan, NQ, NKV, D, True, dev)


def run(mode):
    for l in range(L):
        q, k, v = sets[l % 2]
        if mode == "A":
            qp.prefill_layer(q, k, v, g, NQ, NKV, 0.5, buffers=buf)
        elif mode == "B":
            qp.attention(q, k, v, g, NQ, NKV, out=buf.o)
        else:
            qp.attention(q, k, v, g, NQ, NKV, out=buf.o)
            qp.prune(k, v, g, NKV, D, qp.Scorer.key_norm_small, 0.5)


for rep in range(3):
    for mode in ("A", "B", "C"):
        run(mode)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run(mode)
        b.record()
        torch.cuda.synchronize()
        print(f"rep {rep} mode {mode}: {a.elapsed_time(b) / L:.3f} ms per layer", flush=True)
