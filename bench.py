#!/usr/bin/env python
"""QuickPrefill benchmark: pruned-prefill tokens/s on 1..8 B200s (BASELINE.json metric), one JSON line on rank 0.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--config C4|C2]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Workload (default, BASELINE.json configs[3], "C4" of SURVEY.md §8d — the configuration the metric's "tokens/s at
1/2/4/8 B200" is quoted on): an hour of video at 1 FPS, 3600 frames x 256 tokens = 921,600 tokens in 225 groups of
16 frames (4096 tokens), a Qwen2.5-VL-7B-shaped LLM (28 Q / 4 KV heads, head_dim 128) with ALL 28 layers, key-norm
pruning per KV head at rho 0.5, bf16.  A step = the whole video through every layer: per layer, causal GQA
attention (tcgen05) -> key-norm scores -> top-k -> KV compaction into that layer's persistent cache; for N > 1 each
layer's cache all-gather (one grouped NCCL call through the C ABI, qvk_allgather_layer) runs on a second stream,
overlapped with the next layer.  Strong scaling: the 225 groups are split over the N ranks (qvk_plan_groups).
The projection GEMM is not part of `value` (the north star's five subsystems) — `full_layer` and `e2e`
add it.  `--config C2` runs the round-1 single-layer workload (configs[1]) instead.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import platform
import statistics
import subprocess
import sys
import time
from pathlib import Path


ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    "C4": dict(workload="C4: 1 h video @ 1 FPS (3600 frames x 256 tok = 921,600 tokens, 225 groups of 16 frames), "
                        "qwen2.5-vl-7b shape (28 Q / 4 KV heads, d 128), 28 layers, key-norm rho=0.5 per KV head",
               frames=3600, tokens_per_frame=256, frames_per_group=16, n_q=28, n_kv=4, d_h=128, rho=0.5, layers=28,
               scorer="key_norm_small", pruning="per KV head", scaling="strong"),
    "C2": dict(workload="C2: qwen2.5-vl-7b layer, 256 frames x 256 tok, 16 frames/group, key-norm rho=0.5 per KV head",
               frames=256, tokens_per_frame=256, frames_per_group=16, n_q=28, n_kv=4, d_h=128, rho=0.5, layers=1,
               scorer="key_norm_small", pruning="per KV head", scaling="strong"),
}
METRIC = "pruned-prefill tokens/s"


def config_dict(c: dict, world: int) -> dict:
    """The `config` object of the JSON line — identical in both arms (the driver compares them)."""
    return {"workload": c["workload"], "frames": c["frames"], "tokens_per_frame": c["tokens_per_frame"],
            "frames_per_group": c["frames_per_group"],
            "groups": -(-c["frames"] // c["frames_per_group"]), "tokens": c["frames"] * c["tokens_per_frame"],
            "n_q": c["n_q"], "n_kv": c["n_kv"], "head_dim": c["d_h"], "layers": c["layers"], "rho": c["rho"],
            "scorer": c["scorer"], "pruning": c["pruning"], "parallelism": f"group-sharded x{world}",
            "l2": "inputs larger than L2 (Q+K+V of one layer >> 126 MB)"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-full-layer", action="store_true", help="skip the from-hidden-states layer (projection)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU baseline sample budget")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="C4", help="workload (default C4, the metric's)")
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d["hbm_gbs"], d["bf16_tflops"], d.get("bf16_tflops_sustained"), "measured (MEASURED_PEAKS.json)"
    return 6650.0, 1590.0, 1400.0, "fallback (B200_PROFILING.md)"


def flops_attention(sizes, n_q, d):
    return float(sum(4.0 * d * n_q * n * (n + 1) / 2 for n in sizes))


def bytes_prune(plan, n_kv, d):
    """Algorithmic HBM bytes of the fused prune launch (prune_fused.cu): every K row read once to
    score it, the double score written, then per retained (row, head) the V row read, K and V rows written, idx and
    origin written.  Re-reads of retained K rows (L2 hits) are not credited."""
    T, R = plan.total_tokens, plan.total_rows
    score = T * n_kv * (d * 2 + 8)
    gather = R * n_kv * (3 * d * 2 + 8 + 4)
    return float(score + gather)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms while the timed region runs."""

    FIELDS = "index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, index: int):
        self.proc = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(index)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        rows = [[x.strip() for x in line.split(",")] for line in out.splitlines() if line.strip()]
        rows = [r for r in rows if len(r) >= 9]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[1]) for r in rows]
        mx = max(float(r[2]) for r in rows)
        load = [s for s in sm if s > 0.5 * mx] or sm
        reasons = set()
        for r in rows:
            for name, val in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"),
                                 r[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(rows), "power_w_max": max(float(r[3]) for r in rows if r[3] not in ("[N/A]", ""))}


class NvmlSampler:
    """SM clock and clock-event reasons polled through NVML back to back (~0.25 ms per sample) on a background
    thread started before the warm-up, each sample stamped with the host clock; `window(t0, t1)` keeps the samples
    taken inside the timed region (a C2 step is ~1.7 ms — far below nvidia-smi's 200 ms sampling)."""

    BITS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
            ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
            ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
            ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
            ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, device):
        import threading

        import torch

        self.ok = False
        self.err = ""
        try:
            import pynvml as N

            N.nvmlInit()
            h = None
            try:
                pr = torch.cuda.get_device_properties(device)
                h = N.nvmlDeviceGetHandleByPciBusId(
                    "%08x:%02x:%02x.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id))
            except Exception:
                h = N.nvmlDeviceGetHandleByIndex(torch.device(device).index or 0)
            self.N, self.h = N, h
            self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = repr(e)
            return
        self.rows = []
        self.stop_ev = threading.Event()
        self.th = threading.Thread(target=self._run, daemon=True)
        self.th.start()

    def _run(self):
        N, h = self.N, self.h
        while not self.stop_ev.is_set():
            try:
                c = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append((time.perf_counter(), c, r))
            except Exception as e:  # noqa: BLE001
                self.err = repr(e)
            time.sleep(0.001)  # an NVML query itself takes ~0.1-0.5 ms

    def stop(self):
        if self.ok:
            self.stop_ev.set()
            self.th.join(timeout=5)

    def window(self, t0, t1):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable: " + self.err], "samples": 0}
        rows = [(c, r) for t, c, r in list(self.rows) if t0 <= t <= t1]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0,
                    "note": "no NVML sample inside the timed region" + (": " + self.err if self.err else "")}
        reasons = set()
        for _, r in rows:
            for name, attr in self.BITS:
                if r & getattr(self.N, attr, 0):
                    reasons.add(name)
        sm = [float(c) for c, _ in rows]
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_mhz, "reasons": sorted(reasons),
                "samples": len(rows), "source": "NVML, polled back to back; samples stamped inside the timed region"}


# ------------------------------------------------------------------------------------------------ CPU baseline
def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def cpu_sample(c: dict, seconds: float, cores: int):
    """Bounded CPU sample of the same workload on the host cores, per token through ONE layer: the reference's prune
    path (oracle/_ref = the unmodified reference prune_group per KV-head slice, when built) on one whole 4096-token
    group + the oracle C port's fp64 attention (the reference has no attention code) with OpenMP on all cores over a
    strided sample of that group's query rows.  Returns (seconds per token-layer, kind, description, wall seconds)."""
    import torch  # noqa: F401  (threads)
    from oracle import oracle as O

    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    w0 = time.perf_counter()
    N, n_q, n_kv, d = c["frames_per_group"] * c["tokens_per_frame"], c["n_q"], c["n_kv"], c["d_h"]
    q = O.bf16_to_f32(O.synth_bf16(1, 3, 0, 0, N, n_q, d, False)).reshape(N, n_q, d)
    k = O.bf16_to_f32(O.synth_bf16(1, 1, 0, 0, N, n_kv, d, True)).reshape(N, n_kv, d)
    v = O.bf16_to_f32(O.synth_bf16(1, 2, 0, 0, N, n_kv, d, False)).reshape(N, n_kv, d)
    scale = 1 / math.sqrt(d)
    # probe, then size the strided sample to ~seconds of attention work
    t0 = time.perf_counter()
    _, rows = O.attention_rows(q, k, v, n_q, n_kv, d, scale, 7, 1024)
    probe = time.perf_counter() - t0
    step = max(1, int(1024 * probe / max(1e-3, 0.8 * seconds)))
    t0 = time.perf_counter()
    _, rows = O.attention_rows(q, k, v, n_q, n_kv, d, scale, step // 2, step)
    t_attn = (time.perf_counter() - t0) / rows  # seconds per query token (all heads), unbiased over the group
    kind = "port"
    t0 = time.perf_counter()
    if O.ref is not None:
        O.ref_prune_heads(k, v, None, N, n_kv, d, c["rho"])
        kind = "reference"
    else:
        sc = O.score_norm(k, n_kv, d, True)
        O.select_heads(sc, N, n_kv, O.retained_count(c["rho"], N))
    t_prune = (time.perf_counter() - t0) / N
    desc = (f"1 group x {N} tokens, 1 layer: attention (oracle C port, fp64, OpenMP {cores} threads) on {rows} "
            f"strided query rows (every {step}th) = {t_attn * 1e3:.3f} ms/token; prune "
            f"({'reference prune_group per KV-head slice' if kind == 'reference' else 'oracle port'}, 1 thread) "
            f"= {t_prune * 1e6:.2f} us/token; extrapolated linearly to {c['layers']} layer(s) x "
            f"{c['frames'] * c['tokens_per_frame']} tokens")
    return t_attn + t_prune, kind, desc, time.perf_counter() - w0


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    c = CONFIGS[args.config]
    cores = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_sample(c, 1.0, cores)
    per_tok, walls, descs, kind = [], [], [], "port"
    for _ in range(args.steps):
        sec, kind, desc, wall = cpu_sample(c, 3.0, cores)
        per_tok.append(sec)
        walls.append(wall)
        descs.append(desc)
    sec_tok_layer = statistics.mean(per_tok)
    value = 1.0 / (sec_tok_layer * c["layers"])  # tokens/s through all layers
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(walls),
            "higher_is_better": True, "scaling": c["scaling"], "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_dict(c, args.gpus),
            "extrapolated": True,
            "extrapolation": "each step is a bounded sample (one 4096-token group, one layer); value = 1 / (layers x "
                             "measured seconds per token-layer); ms_per_step = the sample's measured wall time",
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "cpu_model": cpu_model(),
                             "kind": kind, "sample": descs[-1]},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------------------ our arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_2505_16175_b200 as qp

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # Test hook (not used by the driver): QVK_BENCH_SHARE_GPU=1 runs every rank on the visible GPU(s) round-robin
    # over gloo, so the multi-rank path (sharding, cache all-gather, max-over-ranks timing) can be exercised on a
    # 1-GPU box; NCCL refuses two ranks on one device, so there the all-gather is torch's (gloo) broadcasts.
    share = os.environ.get("QVK_BENCH_SHARE_GPU") == "1"
    # Test hook (not used by the driver): QVK_BENCH_FORCE_COMM=1 under torchrun with one rank runs the N > 1 code path
    # (process group, the C ABI's NCCL communicator, per-layer all-gathers on the comm stream, the all-gather report)
    # on a single GPU, where NCCL's collectives degenerate to one rank.
    multi = world > 1 or os.environ.get("QVK_BENCH_FORCE_COMM") == "1"
    if share:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if multi:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    from paper_2505_16175_b200.distributed import NcclComm, allgather_cache, segment_bounds

    c = CONFIGS[args.config]
    n_q, n_kv, d, rho, L = c["n_q"], c["n_kv"], c["d_h"], c["rho"], c["layers"]
    plan = qp.GroupPlan.plan(c["frames"], c["frames_per_group"], c["tokens_per_frame"], rho, world)
    local_plan = plan.shard(rank, world)
    g = local_plan.to(dev)
    gidx0 = int(plan.rank_begin[rank])
    sizes = [int(s) for s in local_plan.sizes]
    unit = n_kv * d
    R = plan.total_rows               # rows of the replicated cache (every rank holds all of them)
    row_base = local_plan.row_base    # this rank's first cache row
    bounds = segment_bounds(plan, world)
    scale = 1 / math.sqrt(d)
    stream = torch.cuda.current_stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    # Inputs: synthetic bf16 Q/K/V in HBM.  The stand-in model's layers are independent (prefill.cpp:185-190), so
    # layer l reads set l % 2 of two distinct sets, each far larger than L2 (C4: 7.2 GB per set per GPU).
    n_sets = 2 if L > 1 else 1
    sets = []
    for s_ in range(n_sets):
        sets.append(tuple(torch.cat([qp.synth_bf16(1, tag, s_, gidx0 + i, n, h, d, tag == 1, dev)
                                     for i, n in enumerate(sizes)]) for tag, h in ((3, n_q), (1, n_kv), (2, n_kv))))
    o = torch.empty_like(sets[0][0])
    scores = torch.empty(max(1, local_plan.total_tokens * n_kv), dtype=torch.float64, device=dev)
    idx = torch.empty(max(1, local_plan.total_rows * n_kv), dtype=torch.int32, device=dev)
    k_cache = torch.empty(L, R * unit, dtype=torch.bfloat16, device=dev)   # the pruned cache of every layer
    v_cache = torch.empty_like(k_cache)
    origin = torch.empty(L, R * n_kv, dtype=torch.int64, device=dev)
    bufs = [qp.LayerBuffers(o, scores, idx, k_cache[l], v_cache[l], origin[l]) for l in range(L)]

    comm = None
    if multi and not share:
        comm = NcclComm()  # the C ABI's communicator (qvk_comm_init over the torch process group's bootstrap)
    comm_stream = torch.cuda.Stream(dev) if multi else None

    def gather_layer(l):
        """Layer l's all-gather on the comm stream, after the layer's kernels (overlaps the next layer)."""
        e = torch.cuda.Event()
        e.record(stream)
        comm_stream.wait_event(e)
        with torch.cuda.stream(comm_stream):
            if comm is not None:
                comm.allgather(k_cache[l], v_cache[l], origin[l], bounds, n_kv, d, comm_stream)
            else:
                allgather_cache([k_cache[l], v_cache[l], origin[l]], bounds, [unit, unit, n_kv])

    def step(do_gather=True):
        for l in range(L):
            q, k, v = sets[l % n_sets]
            # one pruned-prefill layer through the C ABI (qvk_prefill_layer): attention, then the fused prune
            # launched with PDL so its CTAs take the SMs the persistent attention grid releases in its tail
            qp.prefill_layer(q, k, v, g, n_q, n_kv, rho, buffers=bufs[l], cache_row_offset=row_base)
            if multi and do_gather:
                gather_layer(l)
        if multi and do_gather:
            e = torch.cuda.Event()
            e.record(comm_stream)
            stream.wait_event(e)  # the step ends when the replicated cache is complete

    sampler = ClockSampler(local)
    nv = NvmlSampler(dev)  # polling from before the warm-up; only the samples inside the timed region are kept
    for _ in range(args.warmup):
        step()
    if multi:
        dist.barrier()
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    t_start, t_end = ev(), ev()
    t_start.record(stream)
    for _ in range(args.steps):
        step()
    t_end.record(stream)
    torch.cuda.synchronize()
    h1 = time.perf_counter()
    nv.stop()
    nv_clocks = nv.window(h0, h1)
    if multi:
        dist.barrier()
    elapsed_ms = t_start.elapsed_time(t_end)
    clocks = sampler.stop()
    if nv_clocks["samples"] >= 3:
        nv_clocks["nvidia_smi"] = clocks  # the 200 ms nvidia-smi samples over warm-up + timed steps
        clocks = nv_clocks
    else:
        clocks["nvml"] = nv_clocks

    # ---- per-kernel times right after the timed region (serialised, event-timed on the launching stream) ----
    attn_ev, prune_ev = [], []
    for rep in range(max(4, min(args.steps, 10))):
        l = rep % L
        q, k, v = sets[l % n_sets]
        kc = k_cache[l, row_base * unit:]
        vc = v_cache[l, row_base * unit:]
        og = origin[l, row_base * n_kv:]
        a0, a1, p1 = ev(), ev(), ev()
        a0.record(stream)
        qp.attention(q, k, v, g, n_q, n_kv, scale, out=o)
        a1.record(stream)
        qp.lib.qvk_prune(stream.cuda_stream, g.ref, k.data_ptr(), v.data_ptr(), qp._lib.QVK_BF16, n_kv, d,
                         int(qp.Scorer.key_norm_small), rho, None, 0, n_kv, scores.data_ptr(), idx.data_ptr(),
                         kc.data_ptr(), vc.data_ptr(), og.data_ptr())
        p1.record(stream)
        attn_ev.append((a0, a1))
        prune_ev.append((a1, p1))
    torch.cuda.synchronize()

    # ---- N > 1: how much of the per-layer all-gather the overlap hides (SURVEY.md §8e "exposed vs hidden") ----
    ag_report = None
    if multi:
        def timed(fn, reps):
            fn()
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = ev(), ev()
            e0.record(stream)
            for _ in range(reps):
                fn()
            e1.record(stream)
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / reps], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return t.item()

        def gather_all():
            for l in range(L):
                gather_layer(l)
            e = torch.cuda.Event()
            e.record(comm_stream)
            stream.wait_event(e)

        reps = max(1, min(3, args.steps))
        comp_ms = timed(lambda: step(do_gather=False), reps)
        ag_ms = timed(gather_all, reps)
        step_ms = elapsed_ms / args.steps
        exposed = max(0.0, step_ms - comp_ms)
        recv = (plan.total_rows - local_plan.total_rows) * n_kv * (2 * d * 2 + 8) * L
        ag_report = {"allgather_ms_alone": ag_ms, "compute_ms_alone": comp_ms, "step_ms": step_ms,
                     "exposed_ms": exposed, "hidden_frac": (1.0 - exposed / ag_ms) if ag_ms > 0 else None,
                     "bytes_received_per_rank_per_step": recv,
                     "nccl_ctas_and_reserved_sms": (int(os.environ.get("QVK_COMM_CTAS", "8"))
                                                    if comm is not None and world > 1 else 0),
                     "collective": "qvk_allgather_layer (NCCL, C ABI)" if comm is not None else
                                   "torch.distributed broadcasts (gloo, shared-GPU test mode)",
                     "note": "exposed = step - compute-only step (max over ranks); layer l's all-gather runs on a "
                             "second stream while layer l+1 computes"}
    attn_ms = [a.elapsed_time(b) for a, b in attn_ev]
    prune_ms = [a.elapsed_time(b) for a, b in prune_ev]
    el = torch.tensor([elapsed_ms, statistics.mean(attn_ms), statistics.mean(prune_ms)], device=dev)
    if multi:
        dist.all_reduce(el, op=dist.ReduceOp.MAX)
    elapsed_ms, attn_avg, prune_avg = el.tolist()
    total_tokens = plan.total_tokens
    value = total_tokens * args.steps / (elapsed_ms / 1e3)
    step_bytes_in = sum(t.numel() * t.element_size() for t in sets[0]) / 1e6
    del sets
    torch.cuda.empty_cache()

    # ---- the same video from hidden states: per layer the QKV projection GEMM with W_l (key-norm fused) ->
    #      attention -> select + gather.  Distinct synthetic weights per layer, the same tokens X in every layer
    #      (the stand-in model, prefill.cpp:188-189) ----
    full = None
    d_model = n_q * d
    if not args.no_full_layer:
        x = torch.cat([qp.synth_bf16(1, 7, 0, gidx0 + i, n, 1, d_model, False, dev) for i, n in enumerate(sizes)])
        x = x.view(-1, d_model)
        wqkv = torch.stack([(qp.synth_bf16(1, 8, l, 0, (n_q + 2 * n_kv) * d, 1, d_model, False, dev).float()
                             * (1.0 / math.sqrt(d_model))).to(torch.bfloat16).view(-1, d_model) for l in range(L)])
        qkv = (torch.empty(local_plan.total_tokens, n_q, d, dtype=torch.bfloat16, device=dev),
               torch.empty(local_plan.total_tokens, n_kv, d, dtype=torch.bfloat16, device=dev),
               torch.empty(local_plan.total_tokens, n_kv, d, dtype=torch.bfloat16, device=dev))

        def full_step():
            for l in range(L):
                qp.prefill_layer_x(x, wqkv[l], g, n_q, n_kv, d, rho, buffers=bufs[l], qkv=qkv,
                                   cache_row_offset=row_base)
                if multi:
                    gather_layer(l)
            if multi:
                e = torch.cuda.Event()
                e.record(comm_stream)
                stream.wait_event(e)

        f_steps = max(1, min(args.steps, 5))
        for _ in range(max(1, min(args.warmup, 2))):
            full_step()
        torch.cuda.synchronize()
        if multi:
            dist.barrier()
        f0, f1 = ev(), ev()
        f0.record(stream)
        for _ in range(f_steps):
            full_step()
        f1.record(stream)
        torch.cuda.synchronize()
        pj = []
        for l in range(max(3, min(args.steps, 6))):
            a0, a1 = ev(), ev()
            a0.record(stream)
            qp.project_qkv(x, wqkv[l % L], n_q, n_kv, d, g, True, *qkv, scores)
            a1.record(stream)
            pj.append((a0, a1))
        torch.cuda.synchronize()
        t = torch.tensor([f0.elapsed_time(f1), statistics.mean(a.elapsed_time(b) for a, b in pj)], device=dev)
        if multi:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        full_ms, proj_ms = t.tolist()
        proj_fl = 2.0 * local_plan.total_tokens * d_model * (n_q + 2 * n_kv) * d
        full = {"value": total_tokens * f_steps / (full_ms / 1e3), "unit": "tokens/s",
                "ms_per_step": full_ms / f_steps, "steps": f_steps,
                "path": "qvk_prefill_layer_x per layer: hidden states X (T x 3584) -> tcgen05 QKV projection GEMM "
                        "with W_l and the key-norm fused into its epilogue -> attention -> fused select+gather (PDL)",
                "projection": {"kernel": "project_qkv_kernel (tcgen05)", "avg_launch_ms": proj_ms,
                               "flop_per_launch": proj_fl, "achieved_tflops": proj_fl / (proj_ms / 1e3) / 1e12},
                "data": "synthetic X ~ N(0,1), W_l ~ N(0, 1/d_model), bf16"}
        del x, wqkv, qkv
        torch.cuda.empty_cache()

    # ---- e2e: the user's call from host video frames through the public API (FramePrefill), host cache out ----
    e2e = None
    if not args.no_e2e:
        side = 28 * int(round(math.sqrt(c["tokens_per_frame"])))  # 448 x 448 frames: 16 x 16 patches of 28 px
        n_frames = local_plan.total_tokens // c["tokens_per_frame"]
        hframes = torch.empty(n_frames, 3, side, side, dtype=torch.uint8, pin_memory=True)
        hframes.copy_(torch.randint(0, 256, (n_frames, 3, side, side), dtype=torch.uint8,
                                    generator=torch.Generator().manual_seed(rank)))
        embed = ((torch.rand(d_model, 3, generator=torch.Generator().manual_seed(11)) * 2 - 1) / 255).to(dev)
        wqkv = torch.stack([(qp.synth_bf16(1, 8, l, 0, (n_q + 2 * n_kv) * d, 1, d_model, False, dev).float()
                             * (1.0 / math.sqrt(d_model))).to(torch.bfloat16).view(-1, d_model) for l in range(L)])
        chunks = int(os.environ.get("QVK_E2E_CHUNKS", "16" if local_plan.n_groups >= 64 else "4"))
        fp = qp.FramePrefill(local_plan, c["tokens_per_frame"], side, side, embed, wqkv, n_q, n_kv, d, rho, dev,
                             chunks=chunks, cache_rows=R, row_base=row_base)
        # each rank reads back the pruned rows it computed, of every layer (the device all-gather replicates the
        # cache on the GPUs, where the decode step consumes it): pinned host buffers of this rank's rows only (8 ranks
        # x the whole 26.8 GB cache would not fit the host)
        lr = local_plan.total_rows
        out_k = torch.empty(L * lr * unit, dtype=torch.bfloat16, pin_memory=True)
        out_v = torch.empty(L * lr * unit, dtype=torch.bfloat16, pin_memory=True)
        out_o = torch.empty(L * lr * n_kv, dtype=torch.int64, pin_memory=True)

        def gather_f():
            if multi:
                for l in range(L):
                    if comm is not None:
                        comm.allgather(fp.k_cache[l], fp.v_cache[l], fp.origin[l], bounds, n_kv, d, stream)
                    else:
                        allgather_cache([fp.k_cache[l], fp.v_cache[l], fp.origin[l]], bounds, [unit, unit, n_kv])

        e_steps = args.steps
        for _ in range(max(1, min(args.warmup, 2))):
            fp.run(hframes, out_k, out_v, out_o, after_compute=gather_f, join=False, out_local=True)
        fp.join()
        torch.cuda.synchronize()
        if multi:
            dist.barrier()
        e0, e1 = ev(), ev()
        e0.record(stream)
        for _ in range(e_steps):
            fp.run(hframes, out_k, out_v, out_o, after_compute=gather_f, join=False, out_local=True)
        fp.join()  # the last step's readback is inside the timed region
        e1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1)], device=dev)
        if multi:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_f = t.item()
        d2h = local_plan.total_rows * n_kv * (2 * d * 2 + 8) * L
        e2e = {"value": total_tokens * e_steps / (t_f / 1e3), "unit": "tokens/s",
               "h2d_bytes_per_step": hframes.numel() * hframes.element_size(), "d2h_bytes_per_step": d2h,
               "ms_per_step": t_f / e_steps,
               "path": "FramePrefill (public API, pipeline.py): pinned host video frames (%d x 3 x %d x %d uint8) -> "
                       "qvk_tokenize_bf16 once -> per layer qvk_prefill_layer_x (QKV projection GEMM with W_l and the "
                       "fused key-norm, attention, select+gather) -> the pruned cache of all %d layers to pinned host; "
                       "%d group chunks, copies on two streams overlapped with the kernels, consecutive steps chained"
                       % (n_frames, side, side, L, chunks),
               "includes": "frames upload, tokenizer, projection GEMMs (not in `value`), attention, prune, readback"}
        del fp, hframes, wqkv, embed, out_k, out_v, out_o
        torch.cuda.empty_cache()

    hbm, tf_burst, tf_sust, peak_src = peaks()
    fl = flops_attention(sizes, n_q, d)
    achieved = fl / (attn_avg / 1e3) / 1e12
    long_step = elapsed_ms / args.steps > 100.0  # a kernel inside a long, power-capped step: the sustained peak
    tf_peak = tf_sust if (long_step and tf_sust) else tf_burst
    prof = ROOT / "profiles" / f"ncu_attention_{args.config.lower()}_summary.json"
    traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch") if prof.exists() else None
    pb = bytes_prune(local_plan, n_kv, d)
    prof_p = ROOT / "profiles" / f"ncu_prune_{args.config.lower()}_summary.json"
    traffic_p = json.loads(prof_p.read_text()).get("dram_bytes_per_launch") if prof_p.exists() else None
    if full is not None:
        full["projection"]["frac_of_peak"] = full["projection"]["achieved_tflops"] / tf_peak
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
            "scaling": c["scaling"], "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": config_dict(c, world),
            "inputs": "per layer l: synthetic bf16 Q/K/V set l %% 2 (%.0f MB per GPU per set, > L2), generated in HBM "
                      "before timing; %d groups x %d tokens on this rank" % (step_bytes_in, len(sizes), sizes[0]),
            "roofline": {"kernel": "attention_fwd_kernel (tcgen05)", "bound": "tensor", "achieved": achieved,
                         "peak": tf_peak, "unit": "TFLOP/s", "frac": achieved / tf_peak,
                         "frac_of_burst": achieved / tf_burst, "traffic": traffic,
                         "traffic_source": (f"ncu --set full capture, {prof.relative_to(ROOT)} (not measured in this "
                                            "run)") if traffic is not None else None,
                         "peak_source": peak_src + (" sustained (kernel inside a long power-capped step)"
                                                    if tf_peak == tf_sust else " burst"),
                         "flop_per_launch": fl, "avg_launch_ms": attn_avg,
                         "timing": "CUDA events around each launch (one layer over this rank's groups) in a "
                                   "serialised pass right after the timed region"},
            "secondary": {"kernels": "prune_fused_kernel: score+select+gather in one cluster launch (qvk_prune), one "
                                     "layer", "avg_ms": prune_avg,
                          "algorithmic_bytes": pb, "achieved_gbs": pb / (prune_avg / 1e3) / 1e9,
                          "hbm_peak_gbs": hbm, "frac": pb / (prune_avg / 1e3) / 1e9 / hbm, "traffic": traffic_p,
                          "traffic_source": f"ncu capture, {prof_p.relative_to(ROOT)}" if traffic_p else None},
            "clocks": clocks, "e2e": e2e, "gpu_launches": 2 * L * args.steps,
            "allgather": ag_report, "full_layer": full,
        }
        if world == 1 and not args.no_cpu_baseline:
            cores = os.cpu_count() or 1
            sec, kind, desc, _ = cpu_sample(c, args.cpu_seconds, cores)
            line["cpu_baseline"] = {"value": 1.0 / (sec * L), "unit": "tokens/s", "cores": cores,
                                    "cpu_model": cpu_model(), "kind": kind, "sample": desc, "extrapolated": True}
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if multi:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
