"""Host-side mirror of the reference's QuickPrefill interface (/root/reference/proj/include/qv/prefill.hpp) over the
C ABI (include/qvk.h).  Same names, argument meaning and error behaviour as the reference; tensors live in HBM.

Two layers:
  * batched, device-resident GQA path (the north star): GroupPlan / DeviceGroups, attention, score, select, gather,
    prune, snapkv_scores, prefill_layer — one launch covers every group of a layer;
  * reference-API mirror (per token, fp32): score_tokens, retained_count, top_k_indices, prune_group, group_count —
    host arrays in, host arrays out, computed by the same kernels (prefill.cpp:192-282, 325-328).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np
import torch

from . import _lib as L
from ._lib import QvError, check, lib


class Scorer(IntEnum):
    """prefill.hpp:37 plus the SnapKV observation-window scorer of the north star."""
    key_norm_small = 0
    value_norm = 1
    attention_score = 2
    snapkv = 3


def scorer_from_name(name: str) -> Scorer:  # prefill.cpp:69-74
    try:
        return Scorer[name]
    except KeyError:
        raise QvError(f"unknown scorer: {name}") from None


@dataclass
class PruneConfig:  # prefill.hpp:41-46
    scorer: Scorer = Scorer.key_norm_small
    rho: float = 1.0

    def validate(self) -> None:
        check(lib.qvk_validate_rho(C.c_double(self.rho)))


def retained_count(rho: float, token_count: int) -> int:  # prefill.cpp:235-238
    return int(lib.qvk_retained_count(rho, token_count))


def group_count(total_frames: int, frames_per_group: int) -> int:  # prefill.cpp:325-328
    out = C.c_uint64()
    check(lib.qvk_group_count(total_frames, frames_per_group, C.byref(out)))
    return out.value


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


# ---------------------------------------------------------------------------------------------------------------
# (a1) group scheduler
# ---------------------------------------------------------------------------------------------------------------
@dataclass
class GroupPlan:
    """Groups of a frame-token stream: token offsets, retained counts, cache offsets (prefill.cpp:170-183, 235-238)."""
    tok_off: np.ndarray      # int64 [G+1] (local rows of q/k/v)
    keep: np.ndarray         # int64 [G]
    row_off: np.ndarray      # int64 [G+1] (local cache rows)
    first_token: np.ndarray  # uint64 [G] global token id of row 0
    rank_begin: np.ndarray = field(default_factory=lambda: np.zeros(2, np.int32))
    row_base: int = 0        # global cache row of local row 0 (sharded plans)

    @property
    def n_groups(self) -> int:
        return len(self.keep)

    @property
    def total_tokens(self) -> int:
        return int(self.tok_off[-1])

    @property
    def total_rows(self) -> int:
        return int(self.row_off[-1])

    @property
    def sizes(self) -> np.ndarray:
        return np.diff(self.tok_off)

    @classmethod
    def plan(cls, total_frames: int, frames_per_group: int, tokens_per_frame: int, rho: float,
             world: int = 1) -> "GroupPlan":
        n = C.c_uint64()
        check(lib.qvk_plan_groups(total_frames, frames_per_group, tokens_per_frame, rho, world, C.byref(n),
                                  None, None, None, None))
        G = n.value
        tok_off = np.zeros(G + 1, np.int64)
        keep = np.zeros(G, np.int64)
        row_off = np.zeros(G + 1, np.int64)
        rank_begin = np.zeros(world + 1, np.int32)
        check(lib.qvk_plan_groups(total_frames, frames_per_group, tokens_per_frame, rho, world, C.byref(n),
                                  tok_off.ctypes.data, keep.ctypes.data, row_off.ctypes.data,
                                  rank_begin.ctypes.data))
        return cls(tok_off, keep, row_off, tok_off[:-1].astype(np.uint64), rank_begin)

    @classmethod
    def from_sizes(cls, sizes, rho: float, first_tokens=None) -> "GroupPlan":
        sizes = np.asarray(sizes, np.int64)
        tok_off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        keep = np.array([retained_count(rho, int(n)) for n in sizes], np.int64)
        row_off = np.concatenate([[0], np.cumsum(keep)]).astype(np.int64)
        ft = tok_off[:-1].astype(np.uint64) if first_tokens is None else np.asarray(first_tokens, np.uint64)
        return cls(tok_off, keep, row_off, ft)

    def shard(self, rank: int, world: int) -> "GroupPlan":
        """Rank-local plan over groups [rank_begin[rank], rank_begin[rank+1]); cache rows keep global offsets."""
        if len(self.rank_begin) != world + 1:
            raise QvError("plan: built for a different world size")
        a, b = int(self.rank_begin[rank]), int(self.rank_begin[rank + 1])
        tok = self.tok_off[a:b + 1] - self.tok_off[a]
        row = self.row_off[a:b + 1] - self.row_off[a]
        return GroupPlan(tok.astype(np.int64), self.keep[a:b].copy(), row.astype(np.int64),
                         self.first_token[a:b].copy(), self.rank_begin, int(self.row_off[a]))

    def to(self, device) -> "DeviceGroups":
        return DeviceGroups(self, device)


class DeviceGroups:
    """Device copy of a GroupPlan plus the qvk_groups descriptor pointing at it."""

    def __init__(self, plan: GroupPlan, device):
        self.plan = plan
        self.tok_off = torch.from_numpy(plan.tok_off).to(device)
        self.keep = torch.from_numpy(plan.keep).to(device)
        self.row_off = torch.from_numpy(plan.row_off).to(device)
        self.first_token = torch.from_numpy(plan.first_token.astype(np.int64)).to(device)
        sizes = plan.sizes
        self.desc = L.QvkGroups(plan.n_groups, int(sizes.max()) if len(sizes) else 0, plan.total_tokens,
                                plan.total_rows, self.tok_off.data_ptr(), self.keep.data_ptr(),
                                self.row_off.data_ptr(), self.first_token.data_ptr())

    @property
    def ref(self):
        return C.byref(self.desc)


# ---------------------------------------------------------------------------------------------------------------
# batched device path
# ---------------------------------------------------------------------------------------------------------------
def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return L.QVK_F32
    if t.dtype == torch.bfloat16:
        return L.QVK_BF16
    raise QvError(f"unsupported dtype {t.dtype}")


def score(k, v, groups: DeviceGroups, heads: int, width: int, scorer: Scorer, text_query=None,
          n_h: int = 1, out=None) -> torch.Tensor:
    """Scores in (group, head, token) layout, float64 (prefill.cpp:192-233)."""
    out = out if out is not None else torch.empty(groups.plan.total_tokens * heads, dtype=torch.float64,
                                                  device=k.device)
    tq_count = 0 if text_query is None else text_query.numel() // (heads * width)
    check(lib.qvk_score(_stream(), groups.ref, _ptr(k), _ptr(v), _dtype_code(k), heads, width, int(scorer),
                        _ptr(text_query), tq_count, n_h, _ptr(out)))
    return out


def select(scores, groups: DeviceGroups, heads: int, out=None) -> torch.Tensor:
    """Top-k indices per (group, head), ascending, in (cache row, head) layout (prefill.cpp:240-253)."""
    out = out if out is not None else torch.empty(groups.plan.total_rows * heads, dtype=torch.int32,
                                                  device=scores.device)
    check(lib.qvk_select(_stream(), groups.ref, _ptr(scores), heads, _ptr(out)))
    return out


def gather(k, v, groups: DeviceGroups, heads: int, width: int, idx=None, k_cache=None, v_cache=None,
           origin=None, with_origin: bool = True):
    """Compact retained rows into the cache; idx None = rho 1 identity (prefill.cpp:263-280, 304-308)."""
    R = groups.plan.total_rows
    k_cache = k_cache if k_cache is not None else torch.empty(R * heads * width, dtype=k.dtype, device=k.device)
    v_cache = v_cache if v_cache is not None else torch.empty(R * heads * width, dtype=v.dtype, device=v.device)
    if with_origin and origin is None:
        origin = torch.empty(R * heads, dtype=torch.int64, device=k.device)
    check(lib.qvk_gather(_stream(), groups.ref, _ptr(k), _ptr(v), _dtype_code(k), heads, width, _ptr(idx),
                         _ptr(k_cache), _ptr(v_cache), _ptr(origin)))
    return k_cache, v_cache, origin


def select_gather(scores, k, v, groups: DeviceGroups, heads: int, width: int, idx=None, k_cache=None,
                  v_cache=None, origin=None):
    """select -> gather from precomputed scores in one launch (qvk_select_gather; e.g. SnapKV scores)."""
    R = groups.plan.total_rows
    dev = k.device
    k_cache = k_cache if k_cache is not None else torch.empty(R * heads * width, dtype=k.dtype, device=dev)
    v_cache = v_cache if v_cache is not None else torch.empty(R * heads * width, dtype=v.dtype, device=dev)
    origin = origin if origin is not None else torch.empty(R * heads, dtype=torch.int64, device=dev)
    idx = idx if idx is not None else torch.empty(max(1, R * heads), dtype=torch.int32, device=dev)
    check(lib.qvk_select_gather(_stream(), groups.ref, _ptr(scores), _ptr(k), _ptr(v), _dtype_code(k), heads, width,
                                _ptr(idx), _ptr(k_cache), _ptr(v_cache), _ptr(origin)))
    return k_cache, v_cache, origin, idx


def prune(k, v, groups: DeviceGroups, heads: int, width: int, scorer: Scorer, rho: float, text_query=None,
          n_h: int = 1):
    """score -> select -> gather for every group (prune_group batched; prefill.cpp:255-282)."""
    R = groups.plan.total_rows
    dev = k.device
    scores = torch.empty(max(1, groups.plan.total_tokens * heads), dtype=torch.float64, device=dev)
    idx = torch.empty(max(1, R * heads), dtype=torch.int32, device=dev)
    kc = torch.empty(R * heads * width, dtype=k.dtype, device=dev)
    vc = torch.empty(R * heads * width, dtype=v.dtype, device=dev)
    origin = torch.empty(R * heads, dtype=torch.int64, device=dev)
    tq_count = 0 if text_query is None else text_query.numel() // (heads * width)
    check(lib.qvk_prune(_stream(), groups.ref, _ptr(k), _ptr(v), _dtype_code(k), heads, width, int(scorer), rho,
                        _ptr(text_query), tq_count, n_h, _ptr(scores), _ptr(idx), _ptr(kc), _ptr(vc), _ptr(origin)))
    return kc, vc, origin, idx


def attention(q, k, v, groups: DeviceGroups, n_q: int, n_kv: int, scale: float | None = None, out=None):
    """Per-group causal GQA attention, bf16 (tcgen05 kernel)."""
    d = q.shape[-1]
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    out = out if out is not None else torch.empty_like(q)
    check(lib.qvk_attention(_stream(), groups.ref, _ptr(q), _ptr(k), _ptr(v), n_q, n_kv, d, scale, _ptr(out)))
    return out


def snapkv_scores(q, k, groups: DeviceGroups, n_q: int, n_kv: int, window: int = 32, pool: int = 1,
                  scale: float | None = None, out=None, window_stats=None):
    """SnapKV scores per (token, KV head); window_stats (from attention_window_stats): second pass only."""
    d = q.shape[-1]
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    out = out if out is not None else torch.empty(groups.plan.total_tokens * n_kv, dtype=torch.float64,
                                                  device=q.device)
    if window_stats is None:
        check(lib.qvk_snapkv_score(_stream(), groups.ref, _ptr(q), _ptr(k), n_q, n_kv, d, window, pool, scale,
                                   _ptr(out)))
    else:
        check(lib.qvk_snapkv_score_stats(_stream(), groups.ref, _ptr(q), _ptr(k), n_q, n_kv, d, window, pool,
                                         scale, _ptr(window_stats), _ptr(out)))
    return out


def attention_window_stats(q, k, v, groups: DeviceGroups, n_q: int, n_kv: int, window: int = 32,
                           scale: float | None = None, out=None, stats=None):
    """attention() that also returns the softmax statistics (m + log2 l, scaled log2 domain) of every group's last
    `window` query rows, shape (n_groups, n_q, window) fp32 (rows before a group's start are left untouched)."""
    d = q.shape[-1]
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    out = out if out is not None else torch.empty_like(q)
    stats = stats if stats is not None else torch.full((groups.plan.n_groups, n_q, window), float("nan"),
                                                        dtype=torch.float32, device=q.device)
    check(lib.qvk_attention_window_stats(_stream(), groups.ref, _ptr(q), _ptr(k), _ptr(v), n_q, n_kv, d, scale,
                                         _ptr(out), window, _ptr(stats)))
    return out, stats


def text_query_sum(text_query, n_q: int, n_kv: int, out=None) -> torch.Tensor:
    """qbar (n_kv, d_h) fp32: the text queries (T, n_q, d_h) pre-summed over text tokens and the query heads of each KV
    head in double, rounded once (qvk_text_query_sum)."""
    T, d = text_query.shape[0], text_query.shape[-1]
    out = out if out is not None else torch.empty(n_kv, d, dtype=torch.float32, device=text_query.device)
    check(lib.qvk_text_query_sum(_stream(), _ptr(text_query), T, n_q, n_kv, d, _ptr(out)))
    return out


def score_text(k, groups: DeviceGroups, text_query, n_q: int, n_kv: int, per_head: bool = True, qbar=None,
               out=None) -> torch.Tensor:
    """GQA attention_score (prefill.cpp:213-230 on the pre-summed text query, qvk_score_text): float64 scores in the
    (group, head, token) layout; text_query (T, n_q, d_h) fp32 on the device (None -> the reference's error)."""
    d = k.shape[-1]
    heads = n_kv if per_head else 1
    T = 0 if text_query is None else text_query.shape[0]
    out = out if out is not None else torch.empty(max(1, groups.plan.total_tokens * heads), dtype=torch.float64,
                                                  device=k.device)
    check(lib.qvk_score_text(_stream(), groups.ref, _ptr(k), n_q, n_kv, d, int(per_head), _ptr(text_query), T,
                             _ptr(qbar), _ptr(out)))
    return out


def reserve_sms(n: int) -> int:
    """Leave n SMs free of the persistent kernels' grids (qvk_reserve_sms) for work on other streams; returns the
    previous reservation.  Results do not depend on it."""
    prev = C.c_int32(0)
    check(lib.qvk_reserve_sms(int(n), C.byref(prev)))
    return prev.value


def last_prune_route() -> int:
    """Route of this thread's last prune step: 0 fused, 1 separate kernels, 2 rho = 1 identity, 3 select + gather on
    precomputed scores (qvk_last_prune_route)."""
    return int(lib.qvk_last_prune_route())


def _layer_params(n_q, n_kv, d, scorer, per_head, rho, scale, snap_window, snap_pool, text_query):
    tq_count = 0 if text_query is None else int(text_query.shape[0])
    return L.QvkLayerParams(n_q, n_kv, d, int(scorer), int(per_head), rho,
                            1.0 / math.sqrt(d) if scale is None else scale, snap_window, snap_pool,
                            _ptr(text_query), tq_count)


@dataclass
class LayerBuffers:
    """Preallocated outputs/workspace of prefill_layer (reused across steps; no allocation on the hot path)."""
    o: torch.Tensor
    scores: torch.Tensor
    idx: torch.Tensor
    k_cache: torch.Tensor
    v_cache: torch.Tensor
    origin: torch.Tensor

    @classmethod
    def allocate(cls, plan: GroupPlan, n_q: int, n_kv: int, d_h: int, per_head: bool, device,
                 cache_rows: int | None = None) -> "LayerBuffers":
        heads = n_kv if per_head else 1
        width = d_h if per_head else n_kv * d_h
        T, R = plan.total_tokens, plan.total_rows if cache_rows is None else cache_rows
        bf = torch.bfloat16
        return cls(torch.empty(T, n_q, d_h, dtype=bf, device=device),
                   torch.empty(max(1, T * heads), dtype=torch.float64, device=device),
                   torch.empty(max(1, plan.total_rows * heads), dtype=torch.int32, device=device),
                   torch.empty(R * heads * width, dtype=bf, device=device),
                   torch.empty(R * heads * width, dtype=bf, device=device),
                   torch.empty(R * heads, dtype=torch.int64, device=device))


def prefill_layer(q, k, v, groups: DeviceGroups, n_q: int, n_kv: int, rho: float,
                  scorer: Scorer = Scorer.key_norm_small, per_head: bool = True, scale: float | None = None,
                  snap_window: int = 32, snap_pool: int = 1, buffers: LayerBuffers | None = None,
                  cache_row_offset: int = 0, text_query=None) -> LayerBuffers:
    """attention -> score -> select -> gather for one layer and every group of the plan (one qvk call).
    text_query: (T, n_q, d_h) fp32 on the device, for Scorer.attention_score."""
    d = q.shape[-1]
    buf = buffers or LayerBuffers.allocate(groups.plan, n_q, n_kv, d, per_head, q.device)
    heads = n_kv if per_head else 1
    width = d if per_head else n_kv * d
    prm = _layer_params(n_q, n_kv, d, scorer, per_head, rho, scale, snap_window, snap_pool, text_query)
    off = cache_row_offset * heads
    kc = buf.k_cache.data_ptr() + off * width * 2
    vc = buf.v_cache.data_ptr() + off * width * 2
    og = buf.origin.data_ptr() + off * 8
    check(lib.qvk_prefill_layer(_stream(), groups.ref, C.byref(prm), _ptr(q), _ptr(k), _ptr(v), _ptr(buf.o),
                                _ptr(buf.scores), _ptr(buf.idx), kc, vc, og))
    return buf


def project_qkv(x, w, n_q: int, n_kv: int, d_h: int, groups: DeviceGroups | None = None, with_scores: bool = False,
                q=None, k=None, v=None, scores=None):
    """[Q | K | V] = X W^T on the tensor cores (qvk_project_qkv); with_scores: key-norm per (token, KV head) fused
    into the epilogue (needs groups).  Returns q, k, v (and scores)."""
    T, d_model = x.shape[0], x.shape[-1]
    dev = x.device
    q = q if q is not None else torch.empty(T, n_q, d_h, dtype=torch.bfloat16, device=dev)
    k = k if k is not None else torch.empty(T, n_kv, d_h, dtype=torch.bfloat16, device=dev)
    v = v if v is not None else torch.empty(T, n_kv, d_h, dtype=torch.bfloat16, device=dev)
    if with_scores and scores is None:
        scores = torch.empty(max(1, T * n_kv), dtype=torch.float64, device=dev)
    check(lib.qvk_project_qkv(_stream(), _ptr(x), T, d_model, _ptr(w), n_q, n_kv, d_h, _ptr(q), _ptr(k), _ptr(v),
                              groups.ref if groups is not None else None, _ptr(scores) if with_scores else None))
    return (q, k, v, scores) if with_scores else (q, k, v)


def prefill_layer_x(x, w, groups: DeviceGroups, n_q: int, n_kv: int, d_h: int, rho: float,
                    scorer: Scorer = Scorer.key_norm_small, per_head: bool = True, scale: float | None = None,
                    snap_window: int = 32, snap_pool: int = 1, buffers: LayerBuffers | None = None,
                    qkv=None, cache_row_offset: int = 0, text_query=None):
    """Projection -> attention -> prune for one layer from hidden states X (qvk_prefill_layer_x)."""
    T, d_model = x.shape[0], x.shape[-1]
    dev = x.device
    buf = buffers or LayerBuffers.allocate(groups.plan, n_q, n_kv, d_h, per_head, dev)
    if qkv is None:
        qkv = (torch.empty(T, n_q, d_h, dtype=torch.bfloat16, device=dev),
               torch.empty(T, n_kv, d_h, dtype=torch.bfloat16, device=dev),
               torch.empty(T, n_kv, d_h, dtype=torch.bfloat16, device=dev))
    heads = n_kv if per_head else 1
    width = d_h if per_head else n_kv * d_h
    prm = _layer_params(n_q, n_kv, d_h, scorer, per_head, rho, scale, snap_window, snap_pool, text_query)
    off = cache_row_offset * heads
    kc = buf.k_cache.data_ptr() + off * width * 2
    vc = buf.v_cache.data_ptr() + off * width * 2
    og = buf.origin.data_ptr() + off * 8
    check(lib.qvk_prefill_layer_x(_stream(), groups.ref, C.byref(prm), _ptr(x), d_model, _ptr(w), _ptr(qkv[0]),
                                  _ptr(qkv[1]), _ptr(qkv[2]), _ptr(buf.o), _ptr(buf.scores), _ptr(buf.idx), kc, vc, og))
    return buf, qkv


def decode_attention(q, k_cache, v_cache, n_q: int, n_kv: int, scale: float | None = None, with_lse: bool = False,
                     out=None, workspace=None):
    """Attention of query tokens q (n_tq, n_q, d) over one layer's pruned cache (rows, n_kv, d) — the decode-step
    consumer (qvk_decode_attention).  Returns o (and the natural-log LSE per (token, head))."""
    n_tq, d = q.shape[0], q.shape[-1]
    rows = k_cache.numel() // (n_kv * d)
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    need = C.c_size_t(0)
    check(lib.qvk_decode_workspace(n_tq, n_q, n_kv, d, rows, C.byref(need)))
    ws = workspace if workspace is not None and workspace.numel() >= need.value else \
        torch.empty(max(1, need.value), dtype=torch.uint8, device=q.device)
    out = out if out is not None else torch.empty(n_tq, n_q, d, dtype=torch.bfloat16, device=q.device)
    lse = torch.empty(n_tq, n_q, dtype=torch.float32, device=q.device) if with_lse else None
    check(lib.qvk_decode_attention(_stream(), _ptr(q), n_tq, n_q, n_kv, d, _ptr(k_cache), _ptr(v_cache), rows, scale,
                                   _ptr(out), _ptr(lse), _ptr(ws), ws.numel()))
    return (out, lse) if with_lse else out


def tokenize(frames, tokens_per_frame: int, embed, bf16: bool = False, out=None):
    """Stand-in tokenizer on the GPU (prefill.cpp:116-168): frames (F, 3, H, W) uint8, embed (d_model, 3) fp32 ->
    tokens (F * tpf, d_model), fp32 bit-identical to the reference, or those values rounded to bf16."""
    F, _, H, W = frames.shape
    d_model = embed.shape[0]
    out = out if out is not None else torch.empty(F * tokens_per_frame, d_model,
                                                  dtype=torch.bfloat16 if bf16 else torch.float32,
                                                  device=frames.device)
    fn = lib.qvk_tokenize_bf16 if bf16 else lib.qvk_tokenize
    check(fn(_stream(), _ptr(frames), F, W, H, tokens_per_frame, _ptr(embed), d_model, _ptr(out)))
    return out


def prefill_layer_dests(q, k, v, groups: DeviceGroups, n_q: int, n_kv: int, rho: float, peers, buffers: LayerBuffers,
                        scorer: Scorer = Scorer.key_norm_small, scale: float | None = None, cache_row_offset: int = 0):
    """prefill_layer whose compaction writes every retained row into this rank's cache AND every peer's
    (distributed.PeerCache over buffers.k_cache / v_cache / origin) — the all-gather fused into the kernel."""
    d = q.shape[-1]
    prm = _layer_params(n_q, n_kv, d, scorer, True, rho, scale, 32, 1, None)
    off = cache_row_offset * n_kv
    n = len(peers.ptrs[0])
    kcs = (C.c_void_p * n)(*[p + off * d * 2 for p in peers.ptrs[0]])
    vcs = (C.c_void_p * n)(*[p + off * d * 2 for p in peers.ptrs[1]])
    ogs = (C.c_void_p * n)(*[p + off * 8 for p in peers.ptrs[2]])
    check(lib.qvk_prefill_layer_dests(_stream(), groups.ref, C.byref(prm), _ptr(q), _ptr(k), _ptr(v),
                                      _ptr(buffers.o), _ptr(buffers.scores), _ptr(buffers.idx), n, kcs, vcs, ogs))
    return buffers


def synth_bf16(seed: int, tag: int, layer: int, group: int, rows: int, heads: int, width: int,
               head_scale: bool, device="cuda") -> torch.Tensor:
    """Synthetic activations generated in HBM (same bits as oracle qvo_synth_bf16)."""
    out = torch.empty(rows, heads, width, dtype=torch.bfloat16, device=device)
    check(lib.qvk_synth_bf16(_stream(), seed, tag, layer, group, rows, heads, width, int(head_scale), _ptr(out)))
    return out


# ---------------------------------------------------------------------------------------------------------------
# reference-API mirror (per token, fp32, host arrays) — prefill.hpp:105-128
# ---------------------------------------------------------------------------------------------------------------
@dataclass
class PrunedGroup:  # prefill.hpp:120-124
    k: np.ndarray
    v: np.ndarray
    indices: np.ndarray


def _single_group(n: int, keep: int, device) -> DeviceGroups:
    return GroupPlan(np.array([0, n], np.int64), np.array([keep], np.int64), np.array([0, keep], np.int64),
                     np.zeros(1, np.uint64)).to(device)


def score_tokens(k, v, token_count: int, n_h: int, d_h: int, scorer: Scorer, text_query=None,
                 device="cuda") -> np.ndarray:
    k = np.ascontiguousarray(k, np.float32).ravel()
    v = np.ascontiguousarray(v, np.float32).ravel()
    d = n_h * d_h
    if k.size != token_count * d or v.size != token_count * d:
        raise QvError("score: tensor shape mismatch")
    tq = None
    if Scorer(scorer) == Scorer.attention_score:
        if text_query is None or np.size(text_query) == 0:
            raise QvError("attention_score scorer requires a text query")
        if np.size(text_query) % d:
            raise QvError("score: text query shape mismatch")
        tq = torch.from_numpy(np.ascontiguousarray(text_query, np.float32).ravel()).to(device)
    if token_count == 0:
        return np.zeros(0, np.float64)
    g = _single_group(token_count, token_count, device)
    out = score(torch.from_numpy(k).to(device), torch.from_numpy(v).to(device), g, 1, d, Scorer(scorer), tq, n_h)
    return out.cpu().numpy()


def top_k_indices(scores, k: int, device="cuda") -> np.ndarray:
    s = np.ascontiguousarray(scores, np.float64).ravel()
    k = min(int(k), s.size)
    if k == 0:
        return np.zeros(0, np.uint32)
    g = _single_group(s.size, k, device)
    return select(torch.from_numpy(s).to(device), g, 1).cpu().numpy().astype(np.uint32)


def prune_group(k, v, token_count: int, n_h: int, d_h: int, prune_cfg: PruneConfig, text_query=None,
                device="cuda") -> PrunedGroup:
    prune_cfg.validate()
    if token_count == 0:
        raise QvError("prune: empty group")
    d = n_h * d_h
    k = np.ascontiguousarray(k, np.float32).ravel()
    v = np.ascontiguousarray(v, np.float32).ravel()
    if prune_cfg.rho == 1.0 and (k.size != token_count * d or v.size != token_count * d):
        return PrunedGroup(k.copy(), v.copy(), np.arange(token_count, dtype=np.uint32))
    if prune_cfg.rho != 1.0 and (k.size != token_count * d or v.size != token_count * d):
        raise QvError("score: tensor shape mismatch")
    tq = None
    if prune_cfg.rho != 1.0 and prune_cfg.scorer == Scorer.attention_score:
        if text_query is None or np.size(text_query) == 0:
            raise QvError("attention_score scorer requires a text query")
        if np.size(text_query) % d:
            raise QvError("score: text query shape mismatch")
        tq = torch.from_numpy(np.ascontiguousarray(text_query, np.float32).ravel()).to(device)
    kept = retained_count(prune_cfg.rho, token_count)
    g = _single_group(token_count, kept, device)
    kc, vc, origin, idx = prune(torch.from_numpy(k).to(device), torch.from_numpy(v).to(device), g, 1, d,
                                prune_cfg.scorer, prune_cfg.rho, tq, n_h)
    return PrunedGroup(kc.cpu().numpy(), vc.cpu().numpy(), origin.cpu().numpy().astype(np.uint32))
