"""TEST INFRASTRUCTURE ONLY — numpy/ctypes access to the CPU oracle.

  ref   : the compiled, UNMODIFIED reference (oracle/_ref/libqvref_capi.so -> libqvref.so, namespace qvref)
  port  : the C restatement (oracle/build/libqv_oracle.so, see qv_oracle.h), incl. attention / SnapKV

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may import this module.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
P = C.c_void_p


def _np(a):
    return a.ctypes.data_as(P)


class RefError(RuntimeError):
    pass


def _load_ref():
    path = HERE / "_ref" / "libqvref_capi.so"
    if not path.exists():
        return None
    lib = C.CDLL(str(path))
    sig = {
        "qvref_last_error": (C.c_char_p, []),
        "qvref_score_tokens": (C.c_int, [P, C.c_size_t, P, C.c_size_t, C.c_size_t, C.c_uint32, C.c_uint32, C.c_int,
                                         P, C.c_size_t, P]),
        "qvref_retained_count": (C.c_size_t, [C.c_double, C.c_size_t]),
        "qvref_top_k_indices": (C.c_int, [P, C.c_size_t, C.c_size_t, P, C.POINTER(C.c_size_t)]),
        "qvref_prune_group": (C.c_int, [P, C.c_size_t, P, C.c_size_t, C.c_size_t, C.c_uint32, C.c_uint32, C.c_int,
                                        C.c_double, P, C.c_size_t, P, P, P, C.POINTER(C.c_size_t)]),
        "qvref_group_count": (C.c_int, [C.c_uint64, C.c_uint32, C.POINTER(C.c_uint64)]),
        "qvref_patch_grid": (None, [C.c_uint32, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]),
        "qvref_validate_prune": (C.c_int, [C.c_double]),
        "qvref_scorer_from_name": (C.c_int, [C.c_char_p, C.POINTER(C.c_int)]),
        "qvref_splitmix64": (C.c_uint64, [C.POINTER(C.c_uint64)]),
        "qvref_fill_pattern": (None, [C.c_int, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, P]),
        "qvref_model_create": (P, [C.c_uint32] * 6 + [C.c_uint64]),
        "qvref_model_destroy": (None, [P]),
        "qvref_model_text_query": (C.c_size_t, [P, P]),
        "qvref_model_project": (C.c_int, [P, P, C.c_size_t, C.c_uint32, P, P]),
        "qvref_model_tokenize": (C.c_int, [P, P, C.c_size_t, C.c_uint32, C.c_uint32, C.c_uint32, P, P, P, P, P,
                                           C.POINTER(C.c_size_t)]),
        "qvref_prefill_frames": (P, [P, P, C.c_size_t, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, C.c_double]),
        "qvref_cache_destroy": (None, [P]),
        "qvref_cache_layers": (C.c_size_t, [P]),
        "qvref_cache_rows": (C.c_size_t, [P, C.c_size_t]),
        "qvref_cache_groups": (C.c_size_t, [P]),
        "qvref_cache_tokens_seen": (C.c_uint64, [P]),
        "qvref_cache_peak_group_tokens": (C.c_size_t, [P]),
        "qvref_cache_value_bytes": (C.c_uint64, [P]),
        "qvref_cache_copy_layer": (None, [P, C.c_size_t, P, P, P]),
        "qvref_cache_retained_per_group": (None, [P, P]),
    }
    for n, (r, a) in sig.items():
        f = getattr(lib, n)
        f.restype, f.argtypes = r, a
    return lib


def _load_port():
    path = HERE / "build" / "libqv_oracle.so"
    if not path.exists():
        return None
    lib = C.CDLL(str(path))
    sig = {
        "qvo_splitmix64": (C.c_uint64, [C.POINTER(C.c_uint64)]),
        "qvo_stream_seed": (C.c_uint64, [C.c_uint64, C.c_uint32, C.c_uint32]),
        "qvo_seeded_matrix": (None, [C.c_uint64, C.c_uint32, C.c_uint32, C.c_size_t, C.c_double, P]),
        "qvo_synth_bf16": (None, [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64, C.c_size_t, C.c_uint32,
                                  C.c_uint32, C.c_int, P]),
        "qvo_score_norm": (None, [P, C.c_size_t, C.c_uint32, C.c_uint32, C.c_int, P]),
        "qvo_score_attention": (None, [P, C.c_size_t, C.c_uint32, C.c_uint32, P, C.c_size_t, P]),
        "qvo_retained_count": (C.c_size_t, [C.c_double, C.c_size_t]),
        "qvo_top_k": (C.c_size_t, [P, C.c_size_t, C.c_size_t, P]),
        "qvo_select_heads": (C.c_size_t, [P, C.c_size_t, C.c_uint32, C.c_size_t, P]),
        "qvo_gather_heads": (None, [P, C.c_size_t, C.c_uint32, C.c_uint32, P, C.c_size_t, P]),
        "qvo_attention": (None, [P, P, P, C.c_size_t, C.c_uint32, C.c_uint32, C.c_uint32, C.c_double, P]),
        "qvo_attention_rows": (C.c_size_t, [P, P, P, C.c_size_t, C.c_uint32, C.c_uint32, C.c_uint32, C.c_double,
                                            C.c_size_t, C.c_size_t, P]),
        "qvo_snapkv_scores": (None, [P, P, C.c_size_t, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                     C.c_double, P]),
        "qvo_plan_groups": (C.c_uint64, [C.c_uint64, C.c_uint32, C.c_uint32, C.c_double, P, P, P]),
    }
    for n, (r, a) in sig.items():
        f = getattr(lib, n)
        f.restype, f.argtypes = r, a
    return lib


ref = _load_ref()
port = _load_port()


def _ref_check(rc):
    if rc != 0:
        raise RefError(ref.qvref_last_error().decode())


# ---------------------------------------------------------------- the compiled reference (qvref::)
def ref_score_tokens(k, v, n, n_h, d_h, scorer, q=None):
    k = np.ascontiguousarray(k, np.float32).ravel()
    v = np.ascontiguousarray(v, np.float32).ravel()
    qa = np.zeros(0, np.float32) if q is None else np.ascontiguousarray(q, np.float32).ravel()
    out = np.zeros(max(n, 1), np.float64)
    _ref_check(ref.qvref_score_tokens(_np(k), k.size, _np(v), v.size, n, n_h, d_h, int(scorer),
                                      _np(qa) if qa.size else None, qa.size, _np(out)))
    return out[:n]


def ref_top_k(scores, k):
    s = np.ascontiguousarray(scores, np.float64).ravel()
    out = np.zeros(max(1, s.size), np.uint32)
    n = C.c_size_t()
    _ref_check(ref.qvref_top_k_indices(_np(s), s.size, k, _np(out), C.byref(n)))
    return out[: n.value]


def ref_prune_group(k, v, n, n_h, d_h, scorer, rho, q=None):
    k = np.ascontiguousarray(k, np.float32).ravel()
    v = np.ascontiguousarray(v, np.float32).ravel()
    qa = np.zeros(0, np.float32) if q is None else np.ascontiguousarray(q, np.float32).ravel()
    ko = np.zeros(max(1, k.size), np.float32)
    vo = np.zeros(max(1, v.size), np.float32)
    io = np.zeros(max(1, n), np.uint32)
    kept = C.c_size_t()
    _ref_check(ref.qvref_prune_group(_np(k), k.size, _np(v), v.size, n, n_h, d_h, int(scorer), rho,
                                     _np(qa) if qa.size else None, qa.size, _np(ko), _np(vo), _np(io),
                                     C.byref(kept)))
    m = kept.value
    d = n_h * d_h
    if rho == 1.0:
        return ko[: k.size], vo[: v.size], io[:m]
    return ko[: m * d], vo[: m * d], io[:m]


def ref_prune_heads(k, v, scores_unused, n, heads, width, rho):
    """Per-head pruning through the UNMODIFIED reference: prune_group on each head slice with n_h = 1 (key norm)."""
    k = np.asarray(k, np.float32).reshape(n, heads, width)
    v = np.asarray(v, np.float32).reshape(n, heads, width)
    outs = []
    for h in range(heads):
        kk, vv, ii = ref_prune_group(np.ascontiguousarray(k[:, h]), np.ascontiguousarray(v[:, h]), n, 1, width,
                                     0, rho)
        outs.append((kk.reshape(-1, width), vv.reshape(-1, width), ii))
    return outs


def ref_pipeline(pattern, seed, frames, w, h, d_model, n_h, d_h, layers, tpf, text, fpg, scorer, rho):
    """Full reference pipeline: fill_pattern frames -> StandInModel -> tokenize -> prefill.  Returns a dict."""
    px = np.zeros(frames * 3 * w * h, np.uint8)
    for f in range(frames):
        ref.qvref_fill_pattern(pattern, seed, f, w, h, _np(px[f * 3 * w * h:]))
    m = ref.qvref_model_create(d_model, n_h, d_h, layers, tpf, text, seed)
    if not m:
        raise RefError(ref.qvref_last_error().decode())
    c = ref.qvref_prefill_frames(m, _np(px), frames, w, h, fpg, int(scorer), rho)
    if not c:
        ref.qvref_model_destroy(m)
        raise RefError(ref.qvref_last_error().decode())
    out = {"layers": []}
    for l in range(ref.qvref_cache_layers(c)):
        r = ref.qvref_cache_rows(c, l)
        k = np.zeros(r * d_model, np.float32)
        v = np.zeros(r * d_model, np.float32)
        o = np.zeros(r, np.uint64)
        ref.qvref_cache_copy_layer(c, l, _np(k), _np(v), _np(o))
        out["layers"].append((k, v, o))
    rpg = np.zeros(ref.qvref_cache_groups(c), np.uint64)
    ref.qvref_cache_retained_per_group(c, _np(rpg))
    out["retained_per_group"] = rpg
    out["tokens_seen"] = ref.qvref_cache_tokens_seen(c)
    out["peak_group_tokens"] = ref.qvref_cache_peak_group_tokens(c)
    out["value_bytes"] = ref.qvref_cache_value_bytes(c)
    out["pixels"] = px
    ref.qvref_cache_destroy(c)
    ref.qvref_model_destroy(m)
    return out


# ---------------------------------------------------------------- the C restatement (qvo_)
def synth_bf16(seed, tag, layer, group, rows, heads, width, head_scale):
    out = np.zeros(rows * heads * width, np.uint16)
    port.qvo_synth_bf16(seed, tag, layer, group, rows, heads, width, int(head_scale), _np(out))
    return out.reshape(rows, heads, width)


def bf16_to_f32(u16):
    return (np.asarray(u16, np.uint16).astype(np.uint32) << 16).view(np.float32)


def score_norm(x, heads, width, negate):
    x = np.ascontiguousarray(x, np.float32).ravel()
    n = x.size // (heads * width)
    out = np.zeros(max(1, n * heads), np.float64)
    port.qvo_score_norm(_np(x), n, heads, width, int(negate), _np(out))
    return out[: n * heads].reshape(heads, n)


def score_attention(k, n, n_h, d_h, q, text_count):
    k = np.ascontiguousarray(k, np.float32).ravel()
    q = np.ascontiguousarray(q, np.float32).ravel()
    out = np.zeros(max(1, n), np.float64)
    port.qvo_score_attention(_np(k), n, n_h, d_h, _np(q), text_count, _np(out))
    return out[:n]


def top_k(scores, k):
    s = np.ascontiguousarray(scores, np.float64).ravel()
    out = np.zeros(max(1, min(k, s.size)), np.uint32)
    m = port.qvo_top_k(_np(s), s.size, k, _np(out))
    return out[:m]


def retained_count(rho, n):
    return int(port.qvo_retained_count(rho, n))


def select_heads(scores, n, heads, k):
    s = np.ascontiguousarray(scores, np.float64).ravel()
    k = min(k, n)
    idx = np.zeros(max(1, k * heads), np.uint32)
    port.qvo_select_heads(_np(s), n, heads, k, _np(idx))
    return idx[: k * heads].reshape(k, heads)


def gather_heads(x, heads, width, idx):
    x = np.ascontiguousarray(x, np.float32).ravel()
    n = x.size // (heads * width)
    idx = np.ascontiguousarray(idx, np.uint32)
    k = idx.shape[0]
    out = np.zeros(max(1, k * heads * width), np.float32)
    port.qvo_gather_heads(_np(x), n, heads, width, _np(idx), k, _np(out))
    return out[: k * heads * width].reshape(k, heads, width)


def attention(q, k, v, n_q, n_kv, d, scale):
    q = np.ascontiguousarray(q, np.float32)
    k = np.ascontiguousarray(k, np.float32)
    v = np.ascontiguousarray(v, np.float32)
    n = q.size // (n_q * d)
    o = np.zeros(n * n_q * d, np.float64)
    port.qvo_attention(_np(q), _np(k), _np(v), n, n_q, n_kv, d, scale, _np(o))
    return o.reshape(n, n_q, d)


def snapkv_scores(q, k, n_q, n_kv, d, window, pool, scale):
    q = np.ascontiguousarray(q, np.float32)
    k = np.ascontiguousarray(k, np.float32)
    n = q.size // (n_q * d)
    out = np.zeros(max(1, n_kv * n), np.float64)
    port.qvo_snapkv_scores(_np(q), _np(k), n, n_q, n_kv, d, window, pool, scale, _np(out))
    return out[: n_kv * n].reshape(n_kv, n)


def plan_groups(frames, fpg, tpf, rho):
    G = (frames + fpg - 1) // fpg
    tok = np.zeros(G + 1, np.int64)
    keep = np.zeros(max(1, G), np.int64)
    row = np.zeros(G + 1, np.int64)
    port.qvo_plan_groups(frames, fpg, tpf, rho, _np(tok), _np(keep), _np(row))
    return tok, keep[:G], row


def attention_rows(q, k, v, n_q, n_kv, d, scale, row_begin, row_step):
    """Strided row sample of the double attention restatement (CPU baseline); returns (o, rows)."""
    q = np.ascontiguousarray(q, np.float32)
    k = np.ascontiguousarray(k, np.float32)
    v = np.ascontiguousarray(v, np.float32)
    n = q.size // (n_q * d)
    o = np.zeros(n * n_q * d, np.float64)
    rows = port.qvo_attention_rows(_np(q), _np(k), _np(v), n, n_q, n_kv, d, scale, row_begin, row_step, _np(o))
    return o.reshape(n, n_q, d), rows


# ---------------------------------------------------------------- GQA attention_score (qvk.h qvk_score_text)
def text_query_sum(q, n_q, n_kv, d):
    """qbar[h, j] = float32(sum_t sum_{x < n_q/n_kv} double(q[t, h*(n_q/n_kv) + x, j])), t outer, x inner — the text
    query pre-summed over text tokens and the query heads of each KV head (one double rounding per addition, like
    numpy's elementwise add)."""
    q = np.asarray(q, np.float32).reshape(-1, n_q, d)
    gq = n_q // n_kv
    acc = np.zeros((n_kv, d), np.float64)
    for t in range(q.shape[0]):
        qt = q[t].reshape(n_kv, gq, d).astype(np.float64)
        for x in range(gq):
            acc = acc + qt[:, x]
    return acc.astype(np.float32)


def score_text_ref(k, n, n_q, n_kv, d, per_head, qbar, text_count):
    """GQA attention_score through the UNMODIFIED reference: qvref::score_tokens (prefill.cpp:213-230) on the ONE
    pre-summed text-query row (n_h = 1, so its divisor is 1 and the result is the sequential double sum itself),
    per KV-head slice (per_head) or on the flattened n_kv*d row; then divided by T * (n_q/n_kv) or T * n_q.
    Returns (heads, n) float64."""
    k = np.asarray(k, np.float32).reshape(n, n_kv, d)
    qbar = np.asarray(qbar, np.float32).reshape(n_kv, d)
    if per_head:
        div = float(text_count) * float(n_q // n_kv)
        return np.stack([ref_score_tokens(np.ascontiguousarray(k[:, h]), np.ascontiguousarray(k[:, h]), n, 1, d, 2,
                                          qbar[h]) / div for h in range(n_kv)])
    div = float(text_count) * float(n_q)
    flat = np.ascontiguousarray(k.reshape(n, n_kv * d))
    return (ref_score_tokens(flat, flat, n, 1, n_kv * d, 2, qbar.ravel()) / div)[None]
