#!/usr/bin/env python
"""QuickPrefill benchmark: pruned-prefill tokens/s on 1..8 B200s (BASELINE.json metric), one JSON line on rank 0.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Workload (BASELINE.json configs[1]): Qwen2.5-VL-7B-shaped layer (28 Q / 4 KV heads, head_dim 128), 256 frames x 256
tokens per GPU, groups of 16 frames (16 groups x 4096 tokens), key-norm pruning per KV head at rho 0.5, bf16.
A step = one pruned-prefill layer over every group: causal GQA attention (tcgen05) -> key-norm scores -> top-k ->
KV compaction into the persistent cache; for N > 1 followed by the NCCL all-gather (per-rank broadcast) that
assembles the replicated pruned cache.  Weak scaling: each GPU owns 16 groups.  The projection GEMM is not part
of the path; Q/K/V are synthetic bf16 generated in HBM before timing.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path


ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CFG = dict(workload="qwen2.5-vl-7b layer, 256 frames x 256 tok/GPU, 16 frames/group, key-norm rho=0.5 per KV head",
           frames_per_gpu=256, tokens_per_frame=256, frames_per_group=16, n_q=28, n_kv=4, d_h=128, rho=0.5,
           layers=1)
METRIC = "pruned-prefill tokens/s"


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
            time.sleep(0.0002)  # an NVML query itself takes ~0.1-0.5 ms

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
def cpu_sample(seconds: float, cores: int):
    """Bounded CPU sample of the same workload on the host cores: the reference's prune path (oracle/_ref
    prune_group per KV-head slice, when built) + the oracle C port's double attention on a strided row sample of one
    4096-token group (the reference has no attention code).  Returns (tokens/s, kind, description)."""
    import torch  # noqa: F401  (threads)
    from oracle import oracle as O

    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    N, n_q, n_kv, d = CFG["frames_per_group"] * CFG["tokens_per_frame"], CFG["n_q"], CFG["n_kv"], CFG["d_h"]
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
        O.ref_prune_heads(k, v, None, N, n_kv, d, CFG["rho"])
        kind = "reference"
    else:
        sc = O.score_norm(k, n_kv, d, True)
        O.select_heads(sc, N, n_kv, O.retained_count(CFG["rho"], N))
    t_prune = (time.perf_counter() - t0) / N
    tps = 1.0 / (t_attn + t_prune)
    desc = (f"1 group x {N} tokens: attention (oracle C port, fp64, OpenMP {cores} threads) on {rows} strided query "
            f"rows (every {step}th) = {t_attn * 1e3:.2f} ms/token; prune "
            f"({'reference prune_group per KV-head slice' if kind == 'reference' else 'oracle port'}, 1 thread) "
            f"= {t_prune * 1e6:.2f} us/token; tokens/s = 1/(sum)")
    return tps, kind, desc


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_sample(2.0, cores)
    vals, descs, kind = [], [], "port"
    t0 = time.perf_counter()
    for _ in range(args.steps):
        tps, kind, desc = cpu_sample(4.0, cores)
        vals.append(tps)
        descs.append(desc)
    wall = time.perf_counter() - t0
    value = statistics.mean(vals)
    n_tok = CFG["frames_per_gpu"] * CFG["tokens_per_frame"]
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * n_tok / value,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": CFG["workload"], **{k: v for k, v in CFG.items()
                                                                         if k != "workload"}},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": kind, "sample": descs[-1]},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": wall}
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
    # 1-GPU box; NCCL refuses two ranks on one device.
    share = os.environ.get("QVK_BENCH_SHARE_GPU") == "1"
    if share:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    from paper_2505_16175_b200.distributed import allgather_cache, segment_bounds

    c = CFG
    n_q, n_kv, d, rho = c["n_q"], c["n_kv"], c["d_h"], c["rho"]
    plan = qp.GroupPlan.plan(c["frames_per_gpu"] * world, c["frames_per_group"], c["tokens_per_frame"], rho, world)
    local_plan = plan.shard(rank, world)
    g = local_plan.to(dev)
    gidx0 = int(plan.rank_begin[rank])
    sizes = [int(s) for s in local_plan.sizes]
    q = torch.cat([qp.synth_bf16(1, 3, 0, gidx0 + i, n, n_q, d, False, dev) for i, n in enumerate(sizes)])
    k = torch.cat([qp.synth_bf16(1, 1, 0, gidx0 + i, n, n_kv, d, True, dev) for i, n in enumerate(sizes)])
    v = torch.cat([qp.synth_bf16(1, 2, 0, gidx0 + i, n, n_kv, d, False, dev) for i, n in enumerate(sizes)])
    buf = qp.LayerBuffers.allocate(local_plan, n_q, n_kv, d, True, dev, cache_rows=plan.total_rows)
    bounds = segment_bounds(plan, world)
    row_base = local_plan.row_base
    scale = 1 / math.sqrt(d)
    stream = torch.cuda.current_stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    attn_ev, prune_ev = [], []
    unit = n_kv * d

    # N > 1: consecutive steps are consecutive layers with their own caches (two alternating buffers); a layer's
    # cache all-gather runs on NCCL's stream, overlapped with the next layer's compute, and is waited
    # for only before its buffer is reused two steps later and at the end of the timed region.
    bufs = [buf] if world == 1 else [buf, qp.LayerBuffers.allocate(local_plan, n_q, n_kv, d, True, dev,
                                                                   cache_rows=plan.total_rows)]
    pending = [[], []]
    step_no = [0]

    def step():
        i = step_no[0] & 1
        step_no[0] += 1
        b = bufs[i % len(bufs)]
        for w_ in pending[i]:
            w_.wait()
        pending[i] = []
        # one pruned-prefill layer through the C ABI (qvk_prefill_layer): attention, then the fused prune launched
        # with PDL so its CTAs take the SMs the persistent attention grid releases in its tail
        qp.prefill_layer(q, k, v, g, n_q, n_kv, rho, buffers=b, cache_row_offset=row_base)
        if world > 1:
            pending[i] = allgather_cache([b.k_cache, b.v_cache, b.origin], bounds, [unit, unit, n_kv], async_op=True)

    def drain():
        for lst in pending:
            for w_ in lst:
                w_.wait()
            lst.clear()

    def kernel_times(reps: int):
        """Per-kernel event times, kernels serialised (no PDL overlap): the roofline figures."""
        kc = buf.k_cache[row_base * unit:]
        vc = buf.v_cache[row_base * unit:]
        og = buf.origin[row_base * n_kv:]
        for _ in range(reps):
            a0, a1, p1 = ev(), ev(), ev()
            a0.record(stream)
            qp.attention(q, k, v, g, n_q, n_kv, scale, out=buf.o)
            a1.record(stream)
            qp.lib.qvk_prune(stream.cuda_stream, g.ref, k.data_ptr(), v.data_ptr(),
                             qp._lib.QVK_BF16, n_kv, d, int(qp.Scorer.key_norm_small), rho, None, 0, n_kv,
                             buf.scores.data_ptr(), buf.idx.data_ptr(), kc.data_ptr(), vc.data_ptr(), og.data_ptr())
            p1.record(stream)
            attn_ev.append((a0, a1))
            prune_ev.append((a1, p1))

    sampler = ClockSampler(local)
    nv = NvmlSampler(dev)  # polling from before the warm-up; only the samples inside the timed region are kept
    for _ in range(args.warmup):
        step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    t_start, t_end = ev(), ev()
    t_start.record(stream)
    for _ in range(args.steps):
        step()
    drain()  # the last layers' all-gathers complete inside the timed region
    t_end.record(stream)
    torch.cuda.synchronize()
    h1 = time.perf_counter()
    nv.stop()
    nv_clocks = nv.window(h0, h1)
    if world > 1:
        dist.barrier()
    elapsed_ms = t_start.elapsed_time(t_end)
    clocks = sampler.stop()
    if nv_clocks["samples"] >= 3:
        nv_clocks["nvidia_smi"] = clocks  # the 200 ms nvidia-smi samples over warm-up + timed steps
        clocks = nv_clocks
    else:
        clocks["nvml"] = nv_clocks
    # per-kernel times right after the timed region, before the clock probe below heats the GPU further
    kernel_times(max(10, args.steps))
    torch.cuda.synchronize()
    if clocks["samples"] < 3:  # timed region shorter than the sampling period: probe the same step for ~1 s
        sampler = ClockSampler(local)
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < 1.2:
            for _ in range(20):
                step()
            torch.cuda.synchronize()
        nvml_info = clocks.get("nvml")
        clocks = sampler.stop()
        clocks["note"] = "sampled over a 1.2 s run of the same step right after the timed region"
        if nvml_info is not None:
            clocks["nvml"] = nvml_info
    drain()
    # ---- N > 1: how much of the cache all-gather the overlap hides (SURVEY.md §8e "exposed vs hidden") ----
    ag_report = None
    if world > 1:
        def timed(fn):
            for _ in range(2):
                fn()
            drain()
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = ev(), ev()
            e0.record(stream)
            for _ in range(args.steps):
                fn()
            drain()
            e1.record(stream)
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return t.item()

        comp_ms = timed(lambda: qp.prefill_layer(q, k, v, g, n_q, n_kv, rho, buffers=bufs[0],
                                                 cache_row_offset=row_base))
        ag_ms = timed(lambda: allgather_cache([bufs[0].k_cache, bufs[0].v_cache, bufs[0].origin], bounds,
                                              [unit, unit, n_kv]))
        step_ms = elapsed_ms / args.steps
        exposed = max(0.0, step_ms - comp_ms)
        recv = (plan.total_rows - local_plan.total_rows) * n_kv * (2 * d * 2 + 8)
        ag_report = {"allgather_ms_alone": ag_ms, "compute_ms_alone": comp_ms, "step_ms": step_ms,
                     "exposed_ms": exposed, "hidden_frac": (1.0 - exposed / ag_ms) if ag_ms > 0 else None,
                     "bytes_received_per_rank_per_step": recv,
                     "note": "exposed = step - compute-only step (max over ranks); the all-gather of layer l runs on "
                             "NCCL's stream while layer l+1 computes"}
    attn_ms = [a.elapsed_time(b) for a, b in attn_ev]
    prune_ms = [a.elapsed_time(b) for a, b in prune_ev]
    el = torch.tensor([elapsed_ms, statistics.mean(attn_ms), statistics.mean(prune_ms)], device=dev)
    if world > 1:
        dist.all_reduce(el, op=dist.ReduceOp.MAX)
    elapsed_ms, attn_avg, prune_avg = el.tolist()
    total_tokens = plan.total_tokens
    value = total_tokens * args.steps / (elapsed_ms / 1e3)

    # ---- N > 1: the same step with the all-gather fused into the compaction (PeerCache: every rank's prune kernel
    #      stores its retained rows into all ranks' caches over NVLink peer memory; one barrier per step) ----
    fused_ag = None
    if world > 1:
        from paper_2505_16175_b200.distributed import PeerCache

        peers, err = None, None
        try:
            peers = PeerCache([buf.k_cache, buf.v_cache, buf.origin])
        except Exception as e:  # noqa: BLE001
            err = repr(e)[:300]
        ok = torch.tensor([0 if peers is None else 1], device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)  # every rank must have mapped its peers, else all skip together
        try:
            if ok.item() == 0:
                raise RuntimeError(err or "a peer rank could not map the caches")

            def fused_step():
                qp.prefill_layer_dests(q, k, v, g, n_q, n_kv, rho, peers, buf, cache_row_offset=row_base)
                peers.fence(dev)

            for _ in range(args.warmup):
                fused_step()
            dist.barrier()
            torch.cuda.synchronize()
            f0, f1 = ev(), ev()
            f0.record(stream)
            for _ in range(args.steps):
                fused_step()
            f1.record(stream)
            torch.cuda.synchronize()
            t = torch.tensor([f0.elapsed_time(f1)], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            fused_ag = {"value": plan.total_tokens * args.steps / (t.item() / 1e3), "unit": "tokens/s",
                        "ms_per_step": t.item() / args.steps,
                        "path": "qvk_prefill_layer_dests: attention + fused prune whose compaction stores every "
                                "retained row into all %d ranks' caches (CUDA IPC peer pointers over NVLink), then one "
                                "cross-rank barrier; no separate all-gather" % world}
            peers.close()
        except Exception as e:  # noqa: BLE001 — reported, never fatal for the bench line
            fused_ag = {"error": repr(e)[:300]}

    # ---- the same layer from hidden states: QKV projection GEMM (key-norm fused) -> attention -> select+gather ----
    full = None
    if not args.no_full_layer:
        d_model = n_q * d
        x = torch.cat([qp.synth_bf16(1, 7, 0, gidx0 + i, n, 1, d_model, False, dev) for i, n in enumerate(sizes)])
        x = x.view(-1, d_model)
        wqkv = (qp.synth_bf16(1, 8, 0, 0, (n_q + 2 * n_kv) * d, 1, d_model, False, dev).float()
                * (1.0 / math.sqrt(d_model))).to(torch.bfloat16).view(-1, d_model)
        qkv = (torch.empty_like(q), torch.empty_like(k), torch.empty_like(v))

        def full_step():
            qp.prefill_layer_x(x, wqkv, g, n_q, n_kv, d, rho, buffers=buf, qkv=qkv, cache_row_offset=row_base)
            if world > 1:
                allgather_cache([buf.k_cache, buf.v_cache, buf.origin], bounds, [unit, unit, n_kv])

        for _ in range(args.warmup):
            full_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        f0, f1 = ev(), ev()
        f0.record(stream)
        for _ in range(args.steps):
            full_step()
        f1.record(stream)
        torch.cuda.synchronize()
        pj = []
        for _ in range(max(3, args.steps)):
            a0, a1 = ev(), ev()
            a0.record(stream)
            qp.project_qkv(x, wqkv, n_q, n_kv, d, g, True, *qkv, buf.scores)
            a1.record(stream)
            pj.append((a0, a1))
        torch.cuda.synchronize()
        t = torch.tensor([f0.elapsed_time(f1), statistics.mean(a.elapsed_time(b) for a, b in pj)], device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        full_ms, proj_ms = t.tolist()
        proj_fl = 2.0 * plan.total_tokens / world * d_model * (n_q + 2 * n_kv) * d
        full = {"value": plan.total_tokens * args.steps / (full_ms / 1e3), "unit": "tokens/s",
                "ms_per_step": full_ms / args.steps,
                "path": "qvk_prefill_layer_x: hidden states X (T x 3584) -> tcgen05 QKV projection GEMM with the "
                        "key-norm fused into its epilogue -> attention -> fused select+gather (PDL)",
                "projection": {"kernel": "project_qkv_kernel (tcgen05)", "avg_launch_ms": proj_ms,
                               "flop_per_launch": proj_fl, "achieved_tflops": proj_fl / (proj_ms / 1e3) / 1e12},
                "data": "synthetic X ~ N(0,1), W ~ N(0, 1/d_model), bf16"}
        del x, wqkv, qkv

    # ---- e2e through the C ABI with host buffers (H2D of this step's Q/K/V, D2H of the pruned cache) ----
    e2e = e2e_qkv = None
    if not args.no_e2e:
        out_k = torch.empty(buf.k_cache.numel(), dtype=torch.bfloat16).pin_memory()
        out_v = torch.empty_like(out_k).pin_memory()
        out_o = torch.empty(buf.origin.numel(), dtype=torch.int64).pin_memory()

        def timed_steps(fn, join):
            for _ in range(max(1, args.warmup)):
                fn()
            join()
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            e0, e1 = ev(), ev()
            e0.record(stream)
            for _ in range(args.steps):
                fn()
            join()  # the last step's readback is inside the timed region
            e1.record(stream)
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1)], device=dev)
            if world > 1:
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return t.item()

        # each rank reads back the pruned rows it computed (the all-gather replicates the cache on the devices,
        # where the decode step consumes it)
        d2h = local_plan.total_rows * n_kv * (2 * d * 2 + 8)
        # (1) the user's call from video frames (the reference's prefill(model, tokenize(frames), prune) scope):
        #     pinned host uint8 frames -> GPU tokenizer -> QKV projection (key-norm fused) -> attention -> select +
        #     gather -> pruned cache back to pinned host, per 4-group chunk with both copies overlapped
        side = 28 * int(round(math.sqrt(c["tokens_per_frame"])))  # 448 x 448 frames: 16 x 16 patches of 28 px
        n_frames = local_plan.total_tokens // c["tokens_per_frame"]
        hframes = torch.randint(0, 256, (n_frames, 3, side, side), dtype=torch.uint8,
                                generator=torch.Generator().manual_seed(rank)).pin_memory()
        d_model = n_q * d
        embed = ((torch.rand(d_model, 3, generator=torch.Generator().manual_seed(11)) * 2 - 1) / 255).to(dev)
        wqkv = (qp.synth_bf16(1, 8, 0, 0, (n_q + 2 * n_kv) * d, 1, d_model, False, dev).float()
                * (1.0 / math.sqrt(d_model))).to(torch.bfloat16).view(-1, d_model)
        e2e_chunks = os.environ.get("QVK_E2E_CHUNKS", "4")  # dev knob: group chunks of the pipeline (n | taper)
        e2e_chunks = int(e2e_chunks) if e2e_chunks.isdigit() else e2e_chunks
        fp = qp.FramePrefill(local_plan, c["tokens_per_frame"], side, side, embed, wqkv, n_q, n_kv, d, rho, dev,
                             chunks=e2e_chunks, cache_rows=plan.total_rows, row_base=row_base)
        gather_f = (lambda: allgather_cache([fp.k_cache, fp.v_cache, fp.origin], bounds, [unit, unit, n_kv])) \
            if world > 1 else None
        t_f = timed_steps(lambda: fp.run(hframes, out_k, out_v, out_o, after_compute=gather_f, join=False), fp.join)
        e2e = {"value": total_tokens * args.steps / (t_f / 1e3), "unit": "tokens/s",
               "h2d_bytes_per_step": hframes.numel() * hframes.element_size(), "d2h_bytes_per_step": d2h,
               "path": "FramePrefill (public API, pipeline.py): pinned host video frames (%d x 3 x %d x %d uint8) -> "
                       "qvk_tokenize_bf16 -> qvk_prefill_layer_x (QKV projection GEMM with fused key-norm, attention, "
                       "select+gather) -> pruned cache to pinned host; %s group chunks, copies on two streams "
                       "overlapped with the kernels, consecutive steps chained (run(join=False): step i+1's uploads "
                       "overlap step i's kernels and readback)" % (n_frames, side, side, e2e_chunks),
               "includes": "frames upload, tokenizer, projection GEMM (not in `value`), attention, prune, readback"}
        del fp, hframes, wqkv, embed
        # (2) the same step from host Q/K/V (the `value` step's inputs in pinned host memory; PCIe-bound)
        hq, hk, hv = (t.cpu().pin_memory() for t in (q, k, v))
        hp = qp.HostPrefill(local_plan, n_q, n_kv, d, rho, dev, chunks=4, cache_rows=plan.total_rows,
                            row_base=row_base)
        gather = (lambda: allgather_cache([hp.k_cache, hp.v_cache, hp.origin], bounds, [unit, unit, n_kv])) \
            if world > 1 else None
        t_q = timed_steps(lambda: hp.run(hq, hk, hv, out_k, out_v, out_o, after_compute=gather, join=False), hp.join)
        e2e_qkv = {"value": total_tokens * args.steps / (t_q / 1e3), "unit": "tokens/s",
                   "h2d_bytes_per_step": sum(x.numel() * x.element_size() for x in (hq, hk, hv)),
                   "d2h_bytes_per_step": d2h,
                   "path": "HostPrefill: qvk_prefill_layer (C ABI) per 4-group chunk, pinned host Q/K/V in and pruned "
                           "cache out on two copy streams overlapped with the kernels, consecutive steps chained"}

    hbm, tf_burst, tf_sust, peak_src = peaks()
    fl = flops_attention(sizes, n_q, d)
    achieved = fl / (attn_avg / 1e3) / 1e12
    prof = ROOT / "profiles" / "ncu_attention_summary.json"
    traffic = None
    if prof.exists():
        traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")
    pb = bytes_prune(local_plan, n_kv, d)
    prof_p = ROOT / "profiles" / "ncu_prune_summary.json"
    traffic_p = json.loads(prof_p.read_text()).get("dram_bytes_per_launch") if prof_p.exists() else None
    if full is not None:
        full["projection"]["frac_of_peak"] = full["projection"]["achieved_tflops"] / tf_burst
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": c["workload"], "tokens_per_gpu": local_plan.total_tokens,
                       "groups_per_gpu": local_plan.n_groups, "group_tokens": sizes[0], "n_q": n_q, "n_kv": n_kv,
                       "head_dim": d, "rho": rho, "scorer": "key_norm_small", "pruning": "per KV head",
                       "layers": c["layers"], "parallelism": f"group-sharded x{world}" + (
                           ", per-layer cache all-gather (NCCL broadcasts) overlapped with the next layer"
                           if world > 1 else ""),
                       "l2": "inputs larger than L2 (Q+K+V %.0f MB per GPU per step)" %
                             ((q.numel() + k.numel() + v.numel()) * 2 / 1e6)},
            "roofline": {"kernel": "attention_fwd_kernel (tcgen05)", "bound": "tensor", "achieved": achieved,
                         "peak": tf_burst, "unit": "TFLOP/s", "frac": achieved / tf_burst, "traffic": traffic,
                         "peak_source": peak_src + " burst", "flop_per_launch": fl,
                         "avg_launch_ms": attn_avg,
                         "timing": "CUDA events around each launch in a serialised pass of max(10, steps) launches right "
                                   "after the timed region (in the timed steps the prune overlaps the attention tail)"},
            "secondary": {"kernels": "prune_fused_kernel: score+select+gather in one cluster launch (qvk_prune)", "avg_ms": prune_avg,
                          "algorithmic_bytes": pb, "achieved_gbs": pb / (prune_avg / 1e3) / 1e9,
                          "hbm_peak_gbs": hbm, "frac": pb / (prune_avg / 1e3) / 1e9 / hbm, "traffic": traffic_p},
            "clocks": clocks, "e2e": e2e, "e2e_qkv": e2e_qkv, "gpu_launches": 2 * args.steps,
            "allgather": ag_report,
            "full_layer": full, "fused_allgather": fused_ag,
        }
        if world == 1 and not args.no_cpu_baseline:
            cores = os.cpu_count() or 1
            tps, kind, desc = cpu_sample(args.cpu_seconds, cores)
            line["cpu_baseline"] = {"value": tps, "unit": "tokens/s", "cores": cores, "kind": kind, "sample": desc}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
