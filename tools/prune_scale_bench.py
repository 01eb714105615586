#!/usr/bin/env python
"""The prune at the metric's scale (one C4 layer: 225 groups x 4096 tokens, 4 KV heads, d 128) measured alone:
plain reductions over the same K (a bandwidth reference), the standalone key-norm kernel, and the fused prune at
rho 0.5 / 0.125 / ~0 (k = 1: scoring + select only).  Each launch after an L2 flush and a ~100 us sleep kernel (the
flush's dirty lines drain, the launch is queued), median of 10.  A/B: QVK_LIB_PATH=build/ab/<rev>/libqvk.so."""
import sys, statistics, json, torch
sys.path.insert(0, '.')
import paper_2505_16175_b200 as qp
dev = torch.device('cuda:0')
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
G, N, H, D = 225, 4096, 4, 128
k = torch.cat([qp.synth_bf16(1, 1, 0, i, N, H, D, True, dev) for i in range(G)])
v = torch.cat([qp.synth_bf16(1, 2, 0, i, N, H, D, False, dev) for i in range(G)])
def timed(fn, reps=10):
    out = []
    for _ in range(reps):
        flush.zero_(); torch.cuda._sleep(200000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); out.append(a.elapsed_time(b))
    return statistics.median(out)
kb = k.numel() * 2
t = timed(lambda: k.view(torch.int16).amax())
print('torch amax over K', round(t*1e3,1), 'us', round(kb/t/1e6), 'GB/s')
t = timed(lambda: k.view(torch.int64).sum())
print('torch int64 sum over K', round(t*1e3,1), 'us', round(kb/t/1e6), 'GB/s')
for rho in (0.5, 0.125, 1/4096):
    plan = qp.GroupPlan.from_sizes([N]*G, rho); g = plan.to(dev)
    if rho == 0.5:
        sc = torch.empty(G*N*H, dtype=torch.float64, device=dev)
        t = timed(lambda: qp.score(k, v, g, H, D, qp.Scorer.key_norm_small, out=sc))
        print('qvk_score (standalone key-norm)', round(t*1e3,1), 'us', round((kb + G*N*H*8)/t/1e6), 'GB/s')
    t = timed(lambda: qp.prune(k, v, g, H, D, qp.Scorer.key_norm_small, rho))
    R = plan.total_rows
    byt = kb + G*N*H*8 + R*H*(3*D*2 + 12)
    print('fused prune rho', rho, round(t*1e3,1), 'us', round(byt/t/1e6), 'GB/s (alg)', 'score-only bytes/t', round((kb)/t/1e6))
