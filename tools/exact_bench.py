#!/usr/bin/env python
"""Times the drop-in path's pieces on the GPU: the exact fp64 projection (qvk_project_exact) at the 7B shape, the exact
tokenizer, and pageable vs pinned host copies of the same sizes.  One JSON line per item."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2505_16175_b200 as qp  # noqa: E402
from paper_2505_16175_b200._lib import check  # noqa: E402

dev = torch.device("cuda", 0)
s = torch.cuda.current_stream().cuda_stream
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for T, d in ((4096, 3584), (65536, 3584), (65536, 512)):
    x = torch.randn(T, d, device=dev)
    w = torch.randn(d, d, device=dev) / d ** 0.5
    out = torch.empty(T, d, device=dev)
    ms = timed(lambda: check(qp.lib.qvk_project_exact(s, x.data_ptr(), T, d, w.data_ptr(), d, out.data_ptr())))
    dfma = T * d * d
    print(json.dumps({"item": "project_exact", "T": T, "d": d, "ms": ms, "tdfma_per_s": dfma / ms / 1e9}), flush=True)
    ref = (x.double() @ w.double()).float()
    print(json.dumps({"item": "project_exact_vs_fp64_matmul_maxdiff", "v": (ref - out).abs().max().item()}))
    del x, w, out, ref
for nbytes in (59 * 2 ** 20, 940 * 2 ** 20):
    n = nbytes // 4
    dsrc = torch.empty(n, device=dev)
    pg = torch.empty(n)
    pn = torch.empty(n, pin_memory=True)
    for name, h in (("pageable", pg), ("pinned", pn)):
        t0 = time.perf_counter()
        h.copy_(dsrc)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        dsrc.copy_(h)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(json.dumps({"item": f"copy_{name}", "mb": nbytes / 2 ** 20, "d2h_gbs": nbytes / (t1 - t0) / 1e9,
                          "h2d_gbs": nbytes / (t2 - t1) / 1e9}), flush=True)
for nbytes in (59 * 2 ** 20, 940 * 2 ** 20):
    n = nbytes // 4
    dsrc = torch.empty(n, device=dev)
    for touched in (False, True):
        pg = torch.empty(n)
        if touched:
            pg.zero_()
        t0 = time.perf_counter()
        check(qp.lib.qvk_memcpy_d2h_pageable(pg.data_ptr(), dsrc.data_ptr(), nbytes, None))
        t1 = time.perf_counter()
        check(qp.lib.qvk_memcpy_h2d_pageable(dsrc.data_ptr(), pg.data_ptr(), nbytes, None))
        t2 = time.perf_counter()
        print(json.dumps({"item": "staged_pageable", "mb": nbytes / 2 ** 20, "dst_touched": touched,
                          "d2h_gbs": nbytes / (t1 - t0) / 1e9, "h2d_gbs": nbytes / (t2 - t1) / 1e9}), flush=True)
