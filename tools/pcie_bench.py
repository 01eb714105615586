"""Pinned host <-> HBM copy bandwidth on this box (the e2e bound): H2D alone, D2H alone, both at once."""
import json
import torch

n = 256 << 20
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, reps=10):
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    e[0].record(s1)
    e[2].record(s2)
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1):
                d_in.copy_(h_in, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h_out.copy_(d_out, non_blocking=True)
    e[1].record(s1)
    e[3].record(s2)
    torch.cuda.synchronize()
    r = {}
    if h2d:
        r["h2d_gbs"] = n * reps / (e[0].elapsed_time(e[1]) / 1e3) / 1e9
    if d2h:
        r["d2h_gbs"] = n * reps / (e[2].elapsed_time(e[3]) / 1e3) / 1e9
    return r


run(True, True, 2)
print(json.dumps({"h2d_only": run(True, False), "d2h_only": run(False, True), "both": run(True, True)}))
