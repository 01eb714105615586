"""ctypes binding of include/qvk.h (libqvk.so).  Loading fails loudly: there is no CPU fallback for the path."""
from __future__ import annotations

import ctypes as C
import os
import re
from pathlib import Path

LIB_DIR = Path(__file__).resolve().parent / "lib"
HEADER = Path(__file__).resolve().parent.parent / "include" / "qvk.h"

QVK_OK, QVK_E_INVALID, QVK_E_CUDA, QVK_E_UNSUPPORTED = 0, -1, -2, -3
QVK_F32, QVK_BF16 = 0, 1
QVK_KEY_NORM_SMALL, QVK_VALUE_NORM, QVK_ATTENTION_SCORE, QVK_SNAPKV = 0, 1, 2, 3


class QvError(RuntimeError):
    """Mirror of qv::Error (error.hpp:8-10): carries the reference's message verbatim."""


class QvkGroups(C.Structure):
    _fields_ = [
        ("n_groups", C.c_int32),
        ("max_tokens", C.c_int64),
        ("total_tokens", C.c_int64),
        ("total_rows", C.c_int64),
        ("tok_off_d", C.c_void_p),
        ("keep_d", C.c_void_p),
        ("row_off_d", C.c_void_p),
        ("first_token_d", C.c_void_p),
    ]


class QvkLayerParams(C.Structure):
    _fields_ = [
        ("n_q", C.c_int32),
        ("n_kv", C.c_int32),
        ("d_h", C.c_int32),
        ("scorer", C.c_int32),
        ("per_head", C.c_int32),
        ("rho", C.c_double),
        ("scale", C.c_float),
        ("snap_window", C.c_int32),
        ("snap_pool", C.c_int32),
        ("text_query_d", C.c_void_p),
        ("text_count", C.c_int64),
    ]


P = C.c_void_p
I32, I64, U32, U64, SZ, F32, F64 = C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_size_t, C.c_float, C.c_double
GP = C.POINTER(QvkGroups)

_SIGS = {
    "qvk_last_error": (C.c_char_p, []),
    "qvk_version": (C.c_int, []),
    "qvk_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "qvk_malloc": (C.c_int, [C.POINTER(P), SZ]),
    "qvk_free": (C.c_int, [P]),
    "qvk_memcpy_h2d": (C.c_int, [P, P, SZ, P]),
    "qvk_memcpy_d2h": (C.c_int, [P, P, SZ, P]),
    "qvk_stream_sync": (C.c_int, [P]),
    "qvk_memcpy_d2h_pageable": (C.c_int, [P, P, SZ, P]),
    "qvk_memcpy_h2d_pageable": (C.c_int, [P, P, SZ, P]),
    "qvk_group_count": (C.c_int, [U64, U32, C.POINTER(U64)]),
    "qvk_retained_count": (SZ, [F64, SZ]),
    "qvk_validate_rho": (C.c_int, [F64]),
    "qvk_plan_groups": (C.c_int, [U64, U32, U32, F64, I32, C.POINTER(U64), P, P, P, P]),
    "qvk_score": (C.c_int, [P, GP, P, P, C.c_int, I32, I32, I32, P, I64, I32, P]),
    "qvk_text_query_sum": (C.c_int, [P, P, I64, I32, I32, I32, P]),
    "qvk_score_text": (C.c_int, [P, GP, P, I32, I32, I32, I32, P, I64, P, P]),
    "qvk_comm_unique_id": (C.c_int, [P]),
    "qvk_comm_init": (C.c_int, [C.POINTER(P), I32, I32, P]),
    "qvk_comm_init_all": (C.c_int, [P, I32, P]),
    "qvk_comm_wrap": (C.c_int, [C.POINTER(P), P]),
    "qvk_comm_rank": (C.c_int, [P, C.POINTER(I32), C.POINTER(I32)]),
    "qvk_comm_check": (C.c_int, [P]),
    "qvk_comm_destroy": (C.c_int, [P]),
    "qvk_comm_group_start": (C.c_int, []),
    "qvk_comm_group_end": (C.c_int, []),
    "qvk_allgather_layer": (C.c_int, [P, P, P, I32, I32, P, P, P]),
    "qvk_last_prune_route": (C.c_int, []),
    "qvk_reserve_sms": (C.c_int, [C.c_int32, C.POINTER(C.c_int32)]),
    "qvk_ctx_create": (C.c_int, [C.POINTER(P), C.POINTER(QvkLayerParams), I32, P, P]),
    "qvk_ctx_groups": (C.c_int, [P, GP]),
    "qvk_ctx_prefill_layer": (C.c_int, [P, P, P, P, P, P, P, P, P]),
    "qvk_ctx_prefill_layer_x": (C.c_int, [P, P, P, I32, P, P, P, P, P, P, P, P]),
    "qvk_ctx_destroy": (C.c_int, [P]),
    "qvk_peer_barrier": (C.c_int, [P, I32, P, I32, U32, P]),
    "qvk_snapkv_score": (C.c_int, [P, GP, P, P, I32, I32, I32, I32, I32, F32, P]),
    "qvk_snapkv_score_stats": (C.c_int, [P, GP, P, P, I32, I32, I32, I32, I32, F32, P, P]),
    "qvk_select": (C.c_int, [P, GP, P, I32, P]),
    "qvk_gather": (C.c_int, [P, GP, P, P, C.c_int, I32, I32, P, P, P, P]),
    "qvk_select_gather": (C.c_int, [P, GP, P, P, P, C.c_int, I32, I32, P, P, P, P]),
    "qvk_prune": (C.c_int, [P, GP, P, P, C.c_int, I32, I32, I32, F64, P, I64, I32, P, P, P, P, P]),
    "qvk_attention": (C.c_int, [P, GP, P, P, P, I32, I32, I32, F32, P]),
    "qvk_attention_window_stats": (C.c_int, [P, GP, P, P, P, I32, I32, I32, F32, P, I32, P]),
    "qvk_prefill_layer": (C.c_int, [P, GP, C.POINTER(QvkLayerParams), P, P, P, P, P, P, P, P, P]),
    "qvk_project_qkv": (C.c_int, [P, P, I64, I32, P, I32, I32, I32, P, P, P, GP, P]),
    "qvk_prefill_layer_x": (C.c_int, [P, GP, C.POINTER(QvkLayerParams), P, I32, P, P, P, P, P, P, P, P, P, P]),
    "qvk_ipc_get_handle": (C.c_int, [P, P, C.POINTER(U64)]),
    "qvk_ipc_open": (C.c_int, [P, C.POINTER(P)]),
    "qvk_ipc_close": (C.c_int, [P]),
    "qvk_prune_dests": (C.c_int, [P, GP, P, P, I32, I32, I32, F64, P, P, I32, P, P, P]),
    "qvk_prefill_layer_dests": (C.c_int, [P, GP, C.POINTER(QvkLayerParams), P, P, P, P, P, P, I32, P, P, P]),
    "qvk_decode_workspace": (C.c_int, [I32, I32, I32, I32, I64, C.POINTER(SZ)]),
    "qvk_decode_attention": (C.c_int, [P, P, I32, I32, I32, I32, P, P, I64, F32, P, P, P, SZ]),
    "qvk_seeded_matrix": (C.c_int, [P, U64, U32, U32, SZ, F64, P]),
    "qvk_project_exact": (C.c_int, [P, P, I64, I32, P, I32, P]),
    "qvk_tokenize": (C.c_int, [P, P, I64, U32, U32, U32, P, I32, P]),
    "qvk_tokenize_bf16": (C.c_int, [P, P, I64, U32, U32, U32, P, I32, P]),
    "qvk_patch_grid": (None, [U32, C.POINTER(U32), C.POINTER(U32)]),
    "qvk_synth_bf16": (C.c_int, [P, U64, U32, U32, U64, I64, I32, I32, I32, P]),
}


def header_symbols() -> list[str]:
    """Every function the C-ABI header declares (the drop-in boundary's export list)."""
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(qvk_[a-z0-9_]+)\s*\(", text)))


def _load() -> C.CDLL:
    # developer A/B hook: QVK_LIB_PATH points at an alternative build of the same library (tools/ab_build.sh)
    path = Path(os.environ["QVK_LIB_PATH"]) if os.environ.get("QVK_LIB_PATH") else LIB_DIR / "libqvk.so"
    if not path.exists():
        raise ImportError(f"{path} is missing: run `python -m paper_2505_16175_b200.build` (no CPU fallback exists)")
    lib = C.CDLL(str(path))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(rc: int) -> None:
    if rc != QVK_OK:
        raise QvError(lib.qvk_last_error().decode())
