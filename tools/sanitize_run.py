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
# round 2: GQA attention_score (text query), staged pageable copies, the per-video context, the CTA-pair attention,
# SnapKV at the C3b kernel routing limit, the exact projection
tq = torch.randn(5, n_q, d, device=dev)
qp.prefill_layer(q, k, v, g, n_q, n_kv, rho, qp.Scorer.attention_score, True, text_query=tq)
qp.prefill_layer(q, k, v, g, n_q, n_kv, rho, qp.Scorer.attention_score, False, text_query=tq)
qp.prefill_layer(q, k, v, g, n_q, n_kv, 1.0)
import os  # noqa: E402
os.environ["QVK_ATTN_2CTA"] = "1"
qp.attention(q, k, v, g, n_q, n_kv)
del os.environ["QVK_ATTN_2CTA"]
import ctypes as C  # noqa: E402
from paper_2505_16175_b200 import _lib as L  # noqa: E402
from paper_2505_16175_b200._lib import check  # noqa: E402
prm = L.QvkLayerParams(n_q, n_kv, d, 0, 1, rho, 1.0 / math.sqrt(d), 32, 1, None, 0)
ctx = C.c_void_p(0)
tok = plan.tok_off.astype("int64")
check(qp.lib.qvk_ctx_create(C.byref(ctx), C.byref(prm), len(sizes), tok.ctypes.data, None))
buf = qp.LayerBuffers.allocate(plan, n_q, n_kv, d, True, dev)
check(qp.lib.qvk_ctx_prefill_layer(ctx, torch.cuda.current_stream().cuda_stream, q.data_ptr(), k.data_ptr(),
                                   v.data_ptr(), buf.o.data_ptr(), buf.k_cache.data_ptr(), buf.v_cache.data_ptr(),
                                   buf.origin.data_ptr()))
torch.cuda.synchronize()
check(qp.lib.qvk_ctx_destroy(ctx))
import numpy as np  # noqa: E402
hb = np.zeros((6 << 20) + 3, np.uint8)
db = torch.empty(hb.size, dtype=torch.uint8, device=dev)
check(qp.lib.qvk_memcpy_h2d_pageable(db.data_ptr(), hb.ctypes.data, hb.size, None))
check(qp.lib.qvk_memcpy_d2h_pageable(hb.ctypes.data, db.data_ptr(), hb.size, None))
xf = torch.randn(70, 96, device=dev)
wf = torch.randn(96, 96, device=dev)
of = torch.empty(70, 96, device=dev)
check(qp.lib.qvk_project_exact(torch.cuda.current_stream().cuda_stream, xf.data_ptr(), 70, 96, wf.data_ptr(), 96,
                               of.data_ptr()))
# round 2, late: SnapKV windows of several operand blocks (two-pass and pass 2 alone), the attention's window
# statistics, the pass-2 flat (item, key tile) split, the layer path with SnapKV pass 1 from the attention (PDL)
qp.snapkv_scores(q, k, g, n_q, n_kv, 100, 3)
_, st = qp.attention_window_stats(q, k, v, g, n_q, n_kv, 100)
qp.snapkv_scores(q, k, g, n_q, n_kv, 100, 1, window_stats=st)
_, st32 = qp.attention_window_stats(q, k, v, g, n_q, n_kv, 32)
qp.snapkv_scores(q, k, g, n_q, n_kv, 32, 1, window_stats=st32)
qp.prefill_layer(q, k, v, g, n_q, n_kv, rho, qp.Scorer.snapkv, True, snap_window=100, snap_pool=3)
torch.cuda.synchronize()
print("sanitize run ok")
