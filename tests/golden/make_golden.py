"""Generates tests/golden/* from the UNMODIFIED reference (oracle/_ref/libqvref*.so, built from /root/reference by
oracle/Makefile).  Run here (where the reference exists); the fixtures are committed and travel to the GPU box.

    python tests/golden/make_golden.py

Fixtures (all at BASELINE.json configs[0], the reference's CPU-runnable "tiny synthetic" case):
  c1_pipeline.npz   full reference pipeline fill_pattern -> StandInModel -> tokenize -> prefill (per-token pruning,
                    the reference's own semantics) for the gradient / checker / noise patterns and two scorers:
                    origins, retained_per_group, sha256 of the K/V bytes, value_bytes.
  c1_gqa.npz        the GQA variant (4 q / 2 kv heads, d_h 64, 16 frames x 64 tokens, group 4 frames, rho 0.5):
                    synthetic bf16 K/V (oracle qvo_synth_bf16, seed 1) pruned per KV head through the reference
                    (prune_group on each head slice with n_h = 1): retained indices + sha256 of the gathered rows.
  kats.json         SPEC.md known-answer examples evaluated by the reference.
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import oracle as O  # noqa: E402

OUT = Path(__file__).resolve().parent
PATTERNS = {"gradient": 0, "noise": 1, "constant": 2, "checker": 3}
C1 = dict(frames=16, w=64, h=64, d_model=256, n_h=4, d_h=64, layers=1, tpf=64, text=16, fpg=4)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def pipeline_cases():
    cases = []
    for pat in ("gradient", "checker", "noise"):
        for scorer, rho in ((0, 0.5), (2, 0.25), (1, 0.5), (0, 1.0)):
            cases.append((pat, scorer, rho))
    return cases


def main() -> None:
    if O.ref is None:
        raise SystemExit("oracle/_ref is not built (make -C oracle)")
    arrays, meta = {}, []
    for i, (pat, scorer, rho) in enumerate(pipeline_cases()):
        c = C1
        r = O.ref_pipeline(PATTERNS[pat], 1, c["frames"], c["w"], c["h"], c["d_model"], c["n_h"], c["d_h"],
                           c["layers"], c["tpf"], c["text"], c["fpg"], scorer, rho)
        k, v, o = r["layers"][0]
        arrays[f"case{i}_origin"] = o
        arrays[f"case{i}_rpg"] = r["retained_per_group"]
        meta.append(dict(case=i, pattern=pat, scorer=scorer, rho=rho, k_sha=sha(k), v_sha=sha(v),
                         rows=int(o.size), value_bytes=int(r["value_bytes"]), tokens_seen=int(r["tokens_seen"]),
                         peak_group_tokens=int(r["peak_group_tokens"]), **c))
    np.savez_compressed(OUT / "c1_pipeline.npz", meta=json.dumps(meta), **arrays)

    # GQA per-head variant: 4 groups x 256 tokens, 2 KV heads, d_h 64 (K/V tags 1/2, per-group streams)
    G, N, H, D, rho = 4, 256, 2, 64, 0.5
    gq = {}
    for g in range(G):
        kb = O.synth_bf16(1, 1, 0, g, N, H, D, True)
        vb = O.synth_bf16(1, 2, 0, g, N, H, D, False)
        kf, vf = O.bf16_to_f32(kb).reshape(N, H, D), O.bf16_to_f32(vb).reshape(N, H, D)
        outs = O.ref_prune_heads(kf, vf, None, N, H, D, rho)
        for h, (kk, vv, ii) in enumerate(outs):
            gq[f"g{g}_h{h}_idx"] = ii
            gq[f"g{g}_h{h}_k_sha"] = np.frombuffer(bytes.fromhex(sha(kk)), np.uint8)
            gq[f"g{g}_h{h}_v_sha"] = np.frombuffer(bytes.fromhex(sha(vv)), np.uint8)
        gq[f"g{g}_k_sha"] = np.frombuffer(bytes.fromhex(sha(kb)), np.uint8)
    np.savez_compressed(OUT / "c1_gqa.npz", G=G, N=N, H=H, D=D, rho=rho, **gq)

    kats = {
        "key_norm_3_4": O.ref_score_tokens(np.array([3, 4, 0, 0], np.float32), np.zeros(4, np.float32), 2, 1, 2,
                                           0).tolist(),
        "key_norm_3_4_signbit": [int(np.signbit(x)) for x in
                                 O.ref_score_tokens(np.array([3, 4, 0, 0], np.float32), np.zeros(4, np.float32), 2,
                                                    1, 2, 0)],
        "all_zero": O.ref_score_tokens(np.zeros(8, np.float32), np.zeros(8, np.float32), 4, 1, 2, 0).tolist(),
        "topk_1323": O.ref_top_k(np.array([1, 3, 2, 3], np.float64), 2).tolist(),
        "topk_signed_zero": O.ref_top_k(np.array([-0.0, 0.0, -0.0, 0.0]), 2).tolist(),
        "retained": {f"{r},{n}": int(O.ref.qvref_retained_count(r, n)) for r, n in
                     [(0.5, 1), (0.5, 3), (0.5, 5), (0.125, 4), (0.125, 12), (0.1, 4096), (0.3, 10), (1e-9, 100),
                      (0.5, 4096), (0.25, 1024), (1.0, 7)]},
        "group_count_3600_16": O.ref.qvref_group_count and 225,
    }
    import ctypes as C
    gc = C.c_uint64()
    O.ref.qvref_group_count(3600, 16, C.byref(gc))
    kats["group_count_3600_16"] = gc.value
    (OUT / "kats.json").write_text(json.dumps(kats, indent=1) + "\n")
    print("wrote", [p.name for p in OUT.glob("*.npz")], "kats.json")


if __name__ == "__main__":
    main()
