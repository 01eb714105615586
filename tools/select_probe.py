"""Developer probe (not part of the product): select / score kernel latency vs shape (event-timed)."""
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2505_16175_b200 as qp  # noqa: E402

dev = torch.device("cuda", 0)


def t(fn, reps=50):
    """GPU time per call: a spin kernel keeps the GPU busy while the CPU enqueues every call (no launch gaps)."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(50_000_000)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for G, N, heads in [(16, 4096, 4), (1, 4096, 1), (64, 4096, 4), (16, 1024, 4), (4, 16384, 4), (225, 4096, 4)]:
    plan = qp.GroupPlan.from_sizes([N] * G, 0.5)
    g = plan.to(dev)
    s = torch.randn(G * N * heads, dtype=torch.float64, device=dev)
    idx = torch.empty(plan.total_rows * heads, dtype=torch.int32, device=dev)
    print(f"select G={G} N={N} heads={heads}: {t(lambda: qp.select(s, g, heads, out=idx)):.1f} us", flush=True)
sizes = [4096] * 16
plan = qp.GroupPlan.from_sizes(sizes, 0.5)
g = plan.to(dev)
k = torch.cat([qp.synth_bf16(1, 1, 0, i, n, 4, 128, True, dev) for i, n in enumerate(sizes)])
out = torch.empty(65536 * 4, dtype=torch.float64, device=dev)
print("score C2 us", t(lambda: qp.score(k, k, g, 4, 128, qp.Scorer.key_norm_small, out=out)))
print("torch k.sum us", t(lambda: k.sum(dtype=torch.float32)))
print("empty kernel us", t(lambda: out.zero_()))
