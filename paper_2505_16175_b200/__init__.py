"""B200-native (sm_100a) QuickPrefill: group-wise prefill of video-frame tokens with per-group KV-cache pruning.

The compute path is libqvk.so (hand-written CUDA behind include/qvk.h); this package is its host-side mirror of the
reference interface (/root/reference/proj/include/qv/prefill.hpp).  Importing fails loudly when the library has
not been built — there is no CPU fallback.
"""
import sys as _sys
from pathlib import Path as _Path

# `python -m paper_2505_16175_b200.build` imports this package before build.py runs: on a clean checkout libqvk.so
# does not exist yet, so that one command skips loading it (everything else fails loudly without the library).
_BUILDING = ("paper_2505_16175_b200.build" in getattr(_sys, "orig_argv", [])[1:3]
             and not (_Path(__file__).resolve().parent / "lib" / "libqvk.so").exists())
if not _BUILDING:
    from ._lib import QvError, header_symbols, lib  # noqa: F401  (raises ImportError if libqvk.so is missing)
    from .prefill import (  # noqa: F401
        DeviceGroups,
        GroupPlan,
        LayerBuffers,
        PrunedGroup,
        PruneConfig,
        Scorer,
        attention,
        attention_window_stats,
        decode_attention,
        gather,
        group_count,
        last_prune_route,
        reserve_sms,
        prefill_layer,
        prefill_layer_dests,
        prefill_layer_x,
        project_qkv,
        prune,
        prune_group,
        retained_count,
        score,
        score_text,
        score_tokens,
        scorer_from_name,
        select,
        select_gather,
        snapkv_scores,
        synth_bf16,
        text_query_sum,
        tokenize,
        top_k_indices,
    )

    from .pipeline import FramePrefill, HostPrefill, StreamingPrefill  # noqa: F401,E402


__all__ = [n for n in dir() if not n.startswith("_")]
