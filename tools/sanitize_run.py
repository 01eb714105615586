#!/usr/bin/env python
"""Tiny invocation of every kernel of the library, for compute-sanitizer (tools/, not product):
    compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import math
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2505_16175_b200 as qp  # noqa: E402

dev = torch.device("cuda", 0)
sizes, n_q, n_kv, d, rho = [384, 200, 1], 8, 2, 128, 0.5
plan = qp.GroupPlan.from_sizes(sizes, rho)
g = plan.to(dev)
T = sum(sizes)
q = torch.randn(T, n_q, d, device=dev).to(torch.bfloat16)
k = torch.randn(T, n_kv, d, device=dev).to(torch.bfloat16)
v = torch.randn(T, n_kv, d, device=dev).to(torch.bfloat16)
for scorer in (qp.Scorer.key_norm_small, qp.Scorer.snapkv):
    qp.prefill_layer(q, k, v, g, n_q, n_kv, rho, scorer, True)
qp.prefill_layer(q, k, v, g, n_q, n_kv, rho, qp.Scorer.value_norm, False)
sc = qp.score(k, v, g, n_kv, d, qp.Scorer.key_norm_small)
idx = qp.select(sc, g, n_kv)
qp.gather(k, v, g, n_kv, d, idx)
x = torch.randn(T, 512, device=dev).to(torch.bfloat16)
w = (torch.randn((n_q + 2 * n_kv) * d, 512, device=dev) / math.sqrt(512)).to(torch.bfloat16)
qp.project_qkv(x, w, n_q, n_kv, d, g, True)
qp.prefill_layer_x(x, w, g, n_q, n_kv, d, rho)
for n_tq in (1, 40):
    qt = torch.randn(n_tq, n_q, d, device=dev).to(torch.bfloat16)
    qp.decode_attention(qt, k, v, n_q, n_kv, with_lse=True)
fr = torch.randint(0, 256, (4, 3, 64, 64), dtype=torch.uint8, device=dev)
qp.tokenize(fr, 64, torch.rand(256, 3, device=dev) / 255, bf16=True)
torch.cuda.synchronize()
print("sanitize run ok")
