"""Host-buffer prefill: group-chunked pipelining of the host<->device copies with the kernels.

The north-star path consumes Q/K/V that a user may hold in (pinned) host memory.  `HostPrefill.run` streams them in
contiguous chunks of groups: the H2D copy of chunk c+1 (copy stream) and the D2H copy of chunk c-1's pruned cache
(a second copy stream) overlap the kernels of chunk c (the caller's stream), so a step costs about
max(copies, kernels) instead of their sum.  Groups are independent and every chunk writes its pruned
rows at their static global cache offsets (prefill.cpp:235-238), so chunking changes nothing in the result.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np
import torch

from . import _lib as L
from ._lib import check, lib
from .prefill import GroupPlan, Scorer


def chunk_bounds(n_groups: int, chunks) -> np.ndarray:
    """Group boundaries of the pipeline chunks.  `chunks` is a count (equal chunks) or "taper": small chunks at both
    ends (the first chunk's upload and the last chunk's kernels + readback are the parts no other chunk overlaps),
    large ones in the middle — e.g. 16 groups -> 1, 2, 3, 4, 3, 2, 1."""
    G = n_groups
    if chunks == "taper":
        sizes, k = [], 1
        while sum(sizes) + 2 * k <= G:
            sizes = sizes[:len(sizes) // 2] + [k, k] + sizes[len(sizes) // 2:]
            k += 1
        rest = G - sum(sizes)
        if rest:
            sizes.insert(len(sizes) // 2, rest)
        return np.concatenate([[0], np.cumsum(sizes)]).astype(int)
    chunks = max(1, min(int(chunks), G))
    return np.linspace(0, G, chunks + 1).round().astype(int)


class _Pipeline:
    """Chunk pipeline shared by HostPrefill / FramePrefill: per chunk, upload (copy stream h2d) -> kernels (the
    caller's stream) -> readback of the chunk's pruned rows (copy stream d2h).  Dependencies are tracked per chunk
    with events, not per call, so consecutive calls (the layers or videos of a serving loop) overlap too: call i+1's
    upload of chunk c waits only for call i's kernels of chunk c (its input slots are free), and call i+1's kernels
    of chunk c wait only for call i's readback of chunk c (its cache rows are read)."""

    def _init_pipeline(self):
        self.h2d = torch.cuda.Stream(self.dev)
        self.d2h = torch.cuda.Stream(self.dev)
        self._consumed = [None] * len(self.parts)  # main: chunk's kernels done (input slots reusable)
        self._read = [None] * len(self.parts)      # d2h: chunk's cache rows read back
        self._tail = []                            # copy-stream events of the last call not yet joined
        self._chained = False                      # last call ran with join=False

    def join(self, stream=None) -> None:
        """Make `stream` (default: current) wait for the copies of earlier calls.  run(join=True) does this at its
        end, so the stream order covers the host outputs; run(join=False) leaves the last readbacks in flight so
        the next call's uploads and kernels overlap them — call join() (or synchronize) before reading the host
        outputs of the last call.  A call following a join=False call does not order its uploads after the work
        already on the caller's stream (that is the overlap): its host inputs must be ready on the host."""
        s = stream or torch.cuda.current_stream(self.dev)
        for e in self._tail:
            s.wait_event(e)
        self._tail = []

    def _pipeline(self, upload, out_k, out_v, out_o, unit, after_compute, join, out_local=False):
        main = torch.cuda.current_stream(self.dev)
        start = torch.cuda.Event()
        start.record(main)  # inputs / outputs the caller prepared on its stream before this call
        if not self._chained:
            self.h2d.wait_event(start)
        self.d2h.wait_event(start)
        self._chained = not join
        for c, part in enumerate(self.parts):
            r0, r1 = part[2], part[3]
            e_in = torch.cuda.Event()
            with torch.cuda.stream(self.h2d):
                if self._consumed[c] is not None:
                    self.h2d.wait_event(self._consumed[c])
                upload(part)
                e_in.record(self.h2d)
            main.wait_event(e_in)
            if self._read[c] is not None:
                main.wait_event(self._read[c])
            self._layer(part, main)
            self._consumed[c] = torch.cuda.Event()
            self._consumed[c].record(main)
            if out_k is not None:
                self.d2h.wait_event(self._consumed[c])
                base = 0 if out_local else self.row_base  # host outputs sized for this rank's rows only, or global
                a, b = base + r0, base + r1
                L_ = self.k_cache.shape[0]
                ok, ov, oo = out_k.view(L_, -1), out_v.view(L_, -1), out_o.view(L_, -1)
                with torch.cuda.stream(self.d2h):
                    for l in range(L_):  # the chunk's rows of every layer's cache
                        ok[l, a * unit:b * unit].copy_(self.k_cache[l, a * unit:b * unit], non_blocking=True)
                        ov[l, a * unit:b * unit].copy_(self.v_cache[l, a * unit:b * unit], non_blocking=True)
                        oo[l, a * self.n_kv:b * self.n_kv].copy_(self.origin[l, a * self.n_kv:b * self.n_kv],
                                                                 non_blocking=True)
                    self._read[c] = torch.cuda.Event()
                    self._read[c].record(self.d2h)
        if after_compute is not None:
            after_compute()  # e.g. the multi-GPU all-gather: device cache replicated, on the caller's stream
        tail = []
        for s in (self.d2h, self.h2d):
            e = torch.cuda.Event()
            e.record(s)
            tail.append(e)
        self._tail = tail
        if join:
            self.join(main)


class HostPrefill(_Pipeline):
    def __init__(self, plan: GroupPlan, n_q: int, n_kv: int, d_h: int, rho: float, device,
                 scorer: Scorer = Scorer.key_norm_small, chunks: int = 4, cache_rows: int | None = None,
                 row_base: int = 0):
        self.plan, self.n_q, self.n_kv, self.d, self.rho = plan, n_q, n_kv, d_h, rho
        self.dev = torch.device(device)
        G = plan.n_groups
        bounds = chunk_bounds(G, chunks)
        self.parts = []
        for a, b in zip(bounds[:-1], bounds[1:]):
            if b <= a:
                continue
            t0, r0 = int(plan.tok_off[a]), int(plan.row_off[a])
            sub = GroupPlan((plan.tok_off[a:b + 1] - t0).astype(np.int64), plan.keep[a:b].copy(),
                            (plan.row_off[a:b + 1] - r0).astype(np.int64), plan.first_token[a:b].copy())
            self.parts.append((t0, int(plan.tok_off[b]), r0, int(plan.row_off[b]), sub.to(self.dev)))
        T, R = plan.total_tokens, plan.total_rows
        bf = torch.bfloat16
        self.q = torch.empty(T, n_q, d_h, dtype=bf, device=self.dev)
        self.k = torch.empty(T, n_kv, d_h, dtype=bf, device=self.dev)
        self.v = torch.empty(T, n_kv, d_h, dtype=bf, device=self.dev)
        self.o = torch.empty(T, n_q, d_h, dtype=bf, device=self.dev)
        self.scores = torch.empty(max(1, T * n_kv), dtype=torch.float64, device=self.dev)
        self.idx = torch.empty(max(1, R * n_kv), dtype=torch.int32, device=self.dev)
        rows = R if cache_rows is None else cache_rows
        self.k_cache = torch.empty(1, rows * n_kv * d_h, dtype=bf, device=self.dev)  # (layers = 1, cache)
        self.v_cache = torch.empty_like(self.k_cache)
        self.origin = torch.empty(1, rows * n_kv, dtype=torch.int64, device=self.dev)
        self.row_base = row_base
        self.prm = L.QvkLayerParams(n_q, n_kv, d_h, int(scorer), 1, rho, 1.0 / math.sqrt(d_h), 32, 1)
        self._init_pipeline()

    def _layer(self, part, stream):
        t0, t1, r0, r1, g = part
        unit = self.n_kv * self.d
        cr = self.row_base + r0
        check(lib.qvk_prefill_layer(stream.cuda_stream, g.ref, C.byref(self.prm), self.q[t0:t1].data_ptr(),
                                    self.k[t0:t1].data_ptr(), self.v[t0:t1].data_ptr(), self.o[t0:t1].data_ptr(),
                                    self.scores[t0 * self.n_kv:].data_ptr(), self.idx[r0 * self.n_kv:].data_ptr(),
                                    self.k_cache[0, cr * unit:].data_ptr(), self.v_cache[0, cr * unit:].data_ptr(),
                                    self.origin[0, cr * self.n_kv:].data_ptr()))

    def run(self, hq, hk, hv, out_k=None, out_v=None, out_o=None, after_compute=None, join=True):
        """One pruned-prefill layer from host Q/K/V (pinned, (T, heads, d) bf16) into the device cache; optional
        pinned host outputs (full cache size) receive this rank's pruned rows at their global offsets, chunk by
        chunk; `after_compute` (e.g. the multi-GPU all-gather) runs on the device after the last chunk's kernels.
        join=False: see `_Pipeline.join`."""
        unit = self.n_kv * self.d

        def upload(part):
            t0, t1 = part[0], part[1]
            self.q[t0:t1].copy_(hq[t0:t1], non_blocking=True)
            self.k[t0:t1].copy_(hk[t0:t1], non_blocking=True)
            self.v[t0:t1].copy_(hv[t0:t1], non_blocking=True)

        self._pipeline(upload, out_k, out_v, out_o, unit, after_compute, join)


class FramePrefill(_Pipeline):
    """Video frames in host memory -> the pruned KV cache of every layer: the end-to-end path of the reference's
    `prefill(model, tokenize(frames), prune)` (prefill.hpp:86-87, 137-138; prefill.cpp:170-183, 293-323) on the GPU.

    Per chunk of groups (contiguous frames): pinned host frames -> HBM on a copy stream; GPU tokenizer (bf16 tokens,
    qvk_tokenize_bf16) ONCE; then for every layer l — the stand-in projects the same tokens in every layer
    (prefill.cpp:188-189, 298-308) — QKV projection with W_l and the key-norm fused (qvk_project_qkv), attention,
    fused select + gather into layer l's cache (qvk_prefill_layer_x); the chunk's pruned rows of every layer ->
    pinned host on a second copy stream.  Chunk c+1's frames upload and chunk c-1's cache readback overlap chunk c's
    kernels.  Frames are (F, 3, H, W) uint8 (decode.hpp:27-55 FrameBuffer slots), H and W divisible by the patch grid
    of tokens_per_frame (prefill.cpp:116-121).  w_qkv: ((n_q + 2 n_kv) d_h, d_model) for one layer or
    (layers, (n_q + 2 n_kv) d_h, d_model); caches are (layers, rows * n_kv * d_h)."""

    def __init__(self, plan: GroupPlan, tokens_per_frame: int, height: int, width: int, embed, w_qkv, n_q: int,
                 n_kv: int, d_h: int, rho: float, device, chunks: int = 4, cache_rows: int | None = None,
                 row_base: int = 0):
        self.plan, self.tpf, self.n_q, self.n_kv, self.d, self.rho = plan, tokens_per_frame, n_q, n_kv, d_h, rho
        self.dev = torch.device(device)
        self.embed = embed
        self.w = w_qkv if w_qkv.dim() == 3 else w_qkv.unsqueeze(0)
        self.layers = int(self.w.shape[0])
        self.d_model = int(embed.shape[0])
        G = plan.n_groups
        bounds = chunk_bounds(G, chunks)
        self.parts = []
        for a, b in zip(bounds[:-1], bounds[1:]):
            if b <= a:
                continue
            t0, r0 = int(plan.tok_off[a]), int(plan.row_off[a])
            sub = GroupPlan((plan.tok_off[a:b + 1] - t0).astype(np.int64), plan.keep[a:b].copy(),
                            (plan.row_off[a:b + 1] - r0).astype(np.int64), plan.first_token[a:b].copy())
            self.parts.append((t0, int(plan.tok_off[b]), r0, int(plan.row_off[b]), sub.to(self.dev)))
        T, R = plan.total_tokens, plan.total_rows
        if T % tokens_per_frame:
            raise ValueError("plan tokens are not whole frames")
        bf = torch.bfloat16
        self.frames = torch.empty(T // tokens_per_frame, 3, height, width, dtype=torch.uint8, device=self.dev)
        self.x = torch.empty(T, self.d_model, dtype=bf, device=self.dev)
        self.q = torch.empty(T, n_q, d_h, dtype=bf, device=self.dev)
        self.k = torch.empty(T, n_kv, d_h, dtype=bf, device=self.dev)
        self.v = torch.empty(T, n_kv, d_h, dtype=bf, device=self.dev)
        self.o = torch.empty(T, n_q, d_h, dtype=bf, device=self.dev)
        self.scores = torch.empty(max(1, T * n_kv), dtype=torch.float64, device=self.dev)
        self.idx = torch.empty(max(1, R * n_kv), dtype=torch.int32, device=self.dev)
        rows = R if cache_rows is None else cache_rows
        self.k_cache = torch.empty(self.layers, rows * n_kv * d_h, dtype=bf, device=self.dev)
        self.v_cache = torch.empty_like(self.k_cache)
        self.origin = torch.empty(self.layers, rows * n_kv, dtype=torch.int64, device=self.dev)
        self.row_base = row_base
        self.prm = L.QvkLayerParams(n_q, n_kv, d_h, int(Scorer.key_norm_small), 1, rho, 1.0 / math.sqrt(d_h), 32, 1)
        self._init_pipeline()

    def _layer(self, part, stream):
        t0, t1, r0, r1, g = part
        f0, f1 = t0 // self.tpf, t1 // self.tpf
        fr = self.frames[f0:f1]
        check(lib.qvk_tokenize_bf16(stream.cuda_stream, fr.data_ptr(), f1 - f0, fr.shape[3], fr.shape[2], self.tpf,
                                    self.embed.data_ptr(), self.d_model, self.x[t0:t1].data_ptr()))
        unit = self.n_kv * self.d
        cr = self.row_base + r0
        for l in range(self.layers):
            check(lib.qvk_prefill_layer_x(stream.cuda_stream, g.ref, C.byref(self.prm), self.x[t0:t1].data_ptr(),
                                          self.d_model, self.w[l].data_ptr(), self.q[t0:t1].data_ptr(),
                                          self.k[t0:t1].data_ptr(), self.v[t0:t1].data_ptr(),
                                          self.o[t0:t1].data_ptr(), self.scores[t0 * self.n_kv:].data_ptr(),
                                          self.idx[r0 * self.n_kv:].data_ptr(), self.k_cache[l, cr * unit:].data_ptr(),
                                          self.v_cache[l, cr * unit:].data_ptr(),
                                          self.origin[l, cr * self.n_kv:].data_ptr()))

    def run(self, hframes, out_k=None, out_v=None, out_o=None, after_compute=None, join=True, out_local=False):
        """Every layer from pinned host frames (F, 3, H, W) uint8 into the device caches; optional pinned host outputs
        (layers x rows) receive this rank's pruned rows chunk by chunk — at their global cache rows, or from row 0 with
        out_local=True (host buffers sized for this rank's rows only); `after_compute` (e.g. the multi-GPU
        all-gather) runs on the device after the last chunk's kernels.  join=False: see `_Pipeline.join`."""
        def upload(part):
            f0, f1 = part[0] // self.tpf, part[1] // self.tpf
            self.frames[f0:f1].copy_(hframes[f0:f1], non_blocking=True)

        self._pipeline(upload, out_k, out_v, out_o, self.n_kv * self.d, after_compute, join, out_local)


class StreamingPrefill(FramePrefill):
    """The overlap pipeline of the paper (SPEC.md:462-535 `overlap_pipeline`): a producer — e.g. the
    CPU video decoder, whose `IntervalHooks::on_done` (decode.hpp:93-99) marks frames ready — submits each group's
    frames as soon as they are decoded, and the group's upload and kernels are enqueued at once, so decoding group
    g + 1 on the CPU overlaps prefilling group g on the GPU: t_total ~ max(t_dec + t_prefill(last group),
    t_prefill + t_dec(first group)).  Groups may be submitted in any order (every group writes its rows at its static
    cache offset, prefill.cpp:235-238); `finish` reads the cache back once every group has been submitted.

        sp = StreamingPrefill(plan, tpf, H, W, embed, w_qkv, n_q, n_kv, d_h, rho, device)
        for g, frames in decoder:          # frames: pinned (frames_in_group, 3, H, W) uint8
            sp.submit(g, frames)
        sp.finish(out_k, out_v, out_o)
    """

    def __init__(self, plan: GroupPlan, tokens_per_frame: int, height: int, width: int, embed, w_qkv, n_q: int,
                 n_kv: int, d_h: int, rho: float, device, cache_rows: int | None = None, row_base: int = 0):
        super().__init__(plan, tokens_per_frame, height, width, embed, w_qkv, n_q, n_kv, d_h, rho, device,
                         chunks=plan.n_groups, cache_rows=cache_rows, row_base=row_base)
        self.submitted = set()

    def submit(self, group: int, frames) -> None:
        """Enqueue group `group`: its frames (pinned host, the group's frame slots) -> HBM, then its kernels."""
        if group in self.submitted or not 0 <= group < len(self.parts):
            raise ValueError(f"group {group} already submitted or out of range")
        part = self.parts[group]
        t0, t1 = part[0], part[1]
        f0, f1 = t0 // self.tpf, t1 // self.tpf
        if tuple(frames.shape) != tuple(self.frames[f0:f1].shape):
            raise ValueError("frames do not match the group's frame slots")
        main = torch.cuda.current_stream(self.dev)
        e_in = torch.cuda.Event()
        with torch.cuda.stream(self.h2d):
            if self._consumed[group] is not None:  # the previous video's kernels of this group read the slots
                self.h2d.wait_event(self._consumed[group])
            self.frames[f0:f1].copy_(frames, non_blocking=True)
            e_in.record(self.h2d)
        main.wait_event(e_in)
        self._layer(part, main)
        self._consumed[group] = torch.cuda.Event()
        self._consumed[group].record(main)
        self.submitted.add(group)

    def finish(self, out_k=None, out_v=None, out_o=None) -> None:
        if len(self.submitted) != len(self.parts):
            raise ValueError("not every group was submitted")
        if out_k is not None:
            out_k.view(-1).copy_(self.k_cache.view(-1), non_blocking=True)
            out_v.view(-1).copy_(self.v_cache.view(-1), non_blocking=True)
            out_o.view(-1).copy_(self.origin.view(-1), non_blocking=True)
        torch.cuda.current_stream(self.dev).synchronize()
        self.submitted = set()
