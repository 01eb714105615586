"""CPU: pin the oracle.  The C restatement (oracle/qv_oracle.c) must agree bit-for-bit with the compiled, unmodified
reference (oracle/_ref) on every function the reference has, and the golden fixtures must reproduce from the
reference.  Attention / SnapKV (no reference code: "parity unpinned") are checked against torch float64."""
import ctypes as C
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import oracle as O

GOLD = Path(__file__).resolve().parent / "golden"
needs_ref = pytest.mark.skipif(O.ref is None, reason="oracle/_ref not built (needs /root/reference at build time)")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ------------------------------------------------------------------ SPEC known answers
@needs_ref
def test_kats_reference_and_port():
    kats = json.loads((GOLD / "kats.json").read_text())
    s = O.ref_score_tokens(np.array([3, 4, 0, 0], np.float32), np.zeros(4, np.float32), 2, 1, 2, 0)
    assert s.tolist() == kats["key_norm_3_4"] == [-5.0, 0.0]
    assert np.signbit(s[1])  # the reference really yields -0.0 for a zero key
    p = O.score_norm(np.array([3, 4, 0, 0], np.float32), 1, 2, True)[0]
    assert p.tobytes() == s.tobytes()
    assert O.top_k(np.array([1, 3, 2, 3.0]), 2).tolist() == kats["topk_1323"] == [1, 3]
    assert O.top_k(np.array([-0.0, 0.0, -0.0, 0.0]), 2).tolist() == kats["topk_signed_zero"] == [0, 1]
    for key, want in kats["retained"].items():
        rho, n = key.split(",")
        assert O.retained_count(float(rho), int(n)) == want
    assert kats["group_count_3600_16"] == 225


@needs_ref
@pytest.mark.parametrize("n,n_h,d_h", [(1, 1, 1), (7, 1, 3), (64, 4, 16), (300, 2, 64), (129, 8, 128)])
def test_norm_scores_bitexact(n, n_h, d_h):
    rng = np.random.default_rng(n * 31 + d_h)
    k = (rng.standard_normal(n * n_h * d_h) * np.exp(rng.standard_normal(n * n_h * d_h))).astype(np.float32)
    v = rng.standard_normal(n * n_h * d_h).astype(np.float32)
    for scorer, x, neg in ((0, k, True), (1, v, False)):
        ref = O.ref_score_tokens(k, v, n, n_h, d_h, scorer)
        port = O.score_norm(x, 1, n_h * d_h, neg)[0]
        assert ref.tobytes() == port.tobytes()


@needs_ref
@pytest.mark.parametrize("n,n_h,d_h,t", [(5, 1, 4, 1), (64, 4, 16, 8), (100, 2, 32, 3)])
def test_attention_score_bitexact(n, n_h, d_h, t):
    rng = np.random.default_rng(n + t)
    k = rng.standard_normal(n * n_h * d_h).astype(np.float32)
    q = rng.standard_normal(t * n_h * d_h).astype(np.float32)
    ref = O.ref_score_tokens(k, k, n, n_h, d_h, 2, q)
    port = O.score_attention(k, n, n_h, d_h, q, t)
    assert ref.tobytes() == port.tobytes()


@needs_ref
@pytest.mark.parametrize("n", [1, 2, 3, 17, 256, 1000, 4096])
def test_topk_matches_reference_with_ties(n):
    rng = np.random.default_rng(n)
    for trial in range(4):
        s = rng.integers(-3, 4, n).astype(np.float64)  # heavy exact ties
        if trial == 1:
            s = rng.standard_normal(n)
        if trial == 2:
            s = np.where(rng.random(n) < 0.5, -0.0, 0.0)
        for k in sorted({0, 1, n // 3, n // 2, max(0, n - 1), n, n + 5}):
            assert O.top_k(s, k).tolist() == O.ref_top_k(s, k).tolist()


@needs_ref
@pytest.mark.parametrize("rho", [0.125, 0.25, 0.5, 1.0])
def test_prune_group_port_vs_reference(rho):
    n, n_h, d_h = 200, 2, 32
    rng = np.random.default_rng(7)
    k = rng.standard_normal(n * n_h * d_h).astype(np.float32)
    v = rng.standard_normal(n * n_h * d_h).astype(np.float32)
    kr, vr, ir = O.ref_prune_group(k, v, n, n_h, d_h, 0, rho)
    kk = O.retained_count(rho, n)
    assert ir.size == kk
    if rho < 1.0:
        s = O.score_norm(k, 1, n_h * d_h, True)[0]
        idx = O.top_k(s, kk)
        assert idx.tolist() == ir.tolist()
        g = O.gather_heads(k, 1, n_h * d_h, idx.reshape(-1, 1))
        assert g.tobytes() == kr.tobytes()


@needs_ref
def test_per_head_prune_equals_reference_head_slices():
    n, H, D, rho = 256, 2, 64, 0.5
    kb = O.synth_bf16(3, 1, 0, 0, n, H, D, True)
    kf = O.bf16_to_f32(kb).reshape(n, H, D)
    scores = O.score_norm(kf, H, D, True)
    idx = O.select_heads(scores, n, H, O.retained_count(rho, n))
    outs = O.ref_prune_heads(kf, kf, None, n, H, D, rho)
    gathered = O.gather_heads(kf, H, D, idx)
    for h, (kk, _vv, ii) in enumerate(outs):
        assert idx[:, h].tolist() == ii.tolist()
        assert gathered[:, h].tobytes() == kk.tobytes()


@needs_ref
def test_seeded_matrix_and_plan_match_reference():
    # weights: project identity rows through the reference model -> rows of W_K
    d = 16
    m = O.ref.qvref_model_create(d, 1, d, 2, 4, 3, 9)
    eye = np.eye(d, dtype=np.float32)
    k = np.zeros(d * d, np.float32)
    v = np.zeros(d * d, np.float32)
    assert O.ref.qvref_model_project(m, O._np(eye), d, 1, O._np(k), O._np(v)) == 0
    w = np.zeros(d * d, np.float32)
    O.port.qvo_seeded_matrix(9, 1, 1, d * d, 1.0 / np.sqrt(d), O._np(w))
    assert w.tobytes() == k.tobytes()
    O.ref.qvref_model_destroy(m)
    gc = C.c_uint64()
    for frames, fpg in [(16, 4), (17, 4), (1, 1), (3600, 16), (5, 7)]:
        tok, keep, row = O.plan_groups(frames, fpg, 64, 0.5)
        assert O.ref.qvref_group_count(frames, fpg, C.byref(gc)) == 0 and gc.value == len(keep)
        sizes = np.diff(tok)
        assert sizes.sum() == frames * 64 and (sizes[:-1] == fpg * 64).all()
        assert [O.ref.qvref_retained_count(0.5, int(s)) for s in sizes] == keep.tolist()


@needs_ref
@pytest.mark.parametrize("case", range(12))
def test_golden_pipeline_reproduces(case):
    z = np.load(GOLD / "c1_pipeline.npz")
    meta = json.loads(str(z["meta"]))[case]
    r = O.ref_pipeline({"gradient": 0, "noise": 1, "constant": 2, "checker": 3}[meta["pattern"]], 1, meta["frames"],
                       meta["w"], meta["h"], meta["d_model"], meta["n_h"], meta["d_h"], meta["layers"], meta["tpf"],
                       meta["text"], meta["fpg"], meta["scorer"], meta["rho"])
    k, v, o = r["layers"][0]
    assert sha(k) == meta["k_sha"] and sha(v) == meta["v_sha"]
    assert o.tolist() == z[f"case{case}_origin"].tolist()
    assert r["retained_per_group"].tolist() == z[f"case{case}_rpg"].tolist()


def test_golden_gqa_port_pinned():
    """The per-head oracle (C port) reproduces the reference-generated per-head fixture."""
    z = np.load(GOLD / "c1_gqa.npz")
    G, N, H, D, rho = (int(z["G"]), int(z["N"]), int(z["H"]), int(z["D"]), float(z["rho"]))
    for g in range(G):
        kb = O.synth_bf16(1, 1, 0, g, N, H, D, True)
        assert hashlib.sha256(kb.tobytes()).digest() == bytes(z[f"g{g}_k_sha"])
        kf = O.bf16_to_f32(kb).reshape(N, H, D)
        idx = O.select_heads(O.score_norm(kf, H, D, True), N, H, O.retained_count(rho, N))
        for h in range(H):
            assert idx[:, h].tolist() == z[f"g{g}_h{h}_idx"].tolist()


# ------------------------------------------------------------------ unpinned restatements vs torch float64
def _torch_attention(q, k, v, n_q, n_kv, scale):
    n = q.shape[0]
    qt = torch.from_numpy(q).double().permute(1, 0, 2)
    kt = torch.from_numpy(k).double().permute(1, 0, 2).repeat_interleave(n_q // n_kv, 0)
    vt = torch.from_numpy(v).double().permute(1, 0, 2).repeat_interleave(n_q // n_kv, 0)
    s = qt @ kt.transpose(1, 2) * scale
    s = s.masked_fill(torch.triu(torch.ones(n, n, dtype=torch.bool), 1), float("-inf"))
    return (torch.softmax(s, -1) @ vt).permute(1, 0, 2).numpy()


@pytest.mark.parametrize("n,n_q,n_kv,d", [(1, 2, 1, 8), (37, 4, 2, 16), (130, 7, 1, 32)])
def test_attention_restatement_vs_torch(n, n_q, n_kv, d):
    rng = np.random.default_rng(n)
    q = rng.standard_normal((n, n_q, d)).astype(np.float32)
    k = rng.standard_normal((n, n_kv, d)).astype(np.float32)
    v = rng.standard_normal((n, n_kv, d)).astype(np.float32)
    o = O.attention(q, k, v, n_q, n_kv, d, 1 / np.sqrt(d))
    np.testing.assert_allclose(o, _torch_attention(q, k, v, n_q, n_kv, 1 / np.sqrt(d)), rtol=1e-10, atol=1e-12)


@pytest.mark.parametrize("n,w,pool", [(50, 8, 1), (50, 64, 1), (300, 32, 7)])
def test_snapkv_restatement_vs_torch(n, w, pool):
    n_q, n_kv, d = 4, 2, 16
    rng = np.random.default_rng(w + pool)
    q = rng.standard_normal((n, n_q, d)).astype(np.float32)
    k = rng.standard_normal((n, n_kv, d)).astype(np.float32)
    got = O.snapkv_scores(q, k, n_q, n_kv, d, w, pool, 0.25)
    W = min(w, n)
    qt = torch.from_numpy(q).double()
    kt = torch.from_numpy(k).double()
    want = torch.zeros(n_kv, n, dtype=torch.float64)
    for h in range(n_q):
        hk = h // (n_q // n_kv)
        s = (qt[n - W:, h] @ kt[:, hk].T) * 0.25
        pos = torch.arange(n - W, n)[:, None]
        s = s.masked_fill(torch.arange(n)[None, :] > pos, float("-inf"))
        want[hk] += torch.softmax(s, -1).sum(0)
    if pool > 1:
        want = torch.nn.functional.avg_pool1d(want[:, None], pool, 1, pool // 2, count_include_pad=True)[:, 0]
    np.testing.assert_allclose(got, want.numpy(), rtol=1e-10, atol=1e-12)


def test_synth_is_deterministic_and_normalish():
    a = O.synth_bf16(1, 1, 0, 0, 512, 2, 64, False)
    b = O.synth_bf16(1, 1, 0, 0, 512, 2, 64, False)
    assert a.tobytes() == b.tobytes()
    x = O.bf16_to_f32(a)
    assert abs(x.mean()) < 0.02 and abs(x.std() - 1.0) < 0.02
    c = O.synth_bf16(1, 1, 0, 1, 512, 2, 64, False)
    assert a.tobytes() != c.tobytes()


@pytest.mark.skipif(O.ref is None, reason="reference oracle not built")
def test_gqa_attention_score_oracle_pinned():
    """The GQA attention_score oracle (oracle.text_query_sum + score_text_ref, the checker of qvk_score_text): the
    pre-summed query equals a pure-Python loop in the stated order, and the scores through the unmodified reference
    equal the C restatement's attention_score on the same single row, divided by the same divisor."""
    rng = np.random.default_rng(3)
    T, n_q, n_kv, d, n = 3, 4, 2, 8, 17
    q = rng.standard_normal((T, n_q, d)).astype(np.float32)
    k = O.bf16_to_f32(O.synth_bf16(2, 1, 0, 0, n, n_kv, d, True)).reshape(n, n_kv, d)
    qbar = O.text_query_sum(q, n_q, n_kv, d)
    gq = n_q // n_kv
    for h in range(n_kv):
        for j in range(d):
            acc = 0.0
            for t in range(T):
                for x in range(gq):
                    acc += float(q[t, h * gq + x, j])
            assert np.float32(acc) == qbar[h, j]
    per_head = O.score_text_ref(k, n, n_q, n_kv, d, True, qbar, T)
    for h in range(n_kv):
        port = O.score_attention(np.ascontiguousarray(k[:, h]), n, 1, d, qbar[h], 1)
        assert np.array_equal(per_head[h], port / (T * gq))
    per_tok = O.score_text_ref(k, n, n_q, n_kv, d, False, qbar, T)
    port = O.score_attention(k.reshape(n, -1), n, 1, n_kv * d, qbar.ravel(), 1)
    assert np.array_equal(per_tok[0], port / (T * n_q))


def test_error_bounded_tie_check():
    """tests/tiecheck.py: swaps within 2 eps of the k-th score pass, a swap outside it and a set that is not the
    top-k of its own scores fail."""
    import pytest as _pt
    from tiecheck import error_bounded_ties
    want = np.array([5.0, 4.0, 3.0, 2.999, 1.0])
    got = want + np.array([0, 0, -0.001, 0.001, 0])        # eps 1e-3: indices 2 and 3 swap (gap 1e-3 <= 2 eps)
    nd, eps, _ = error_bounded_ties([0, 1, 3], got, want, 3)
    assert nd == 2 and abs(eps - 1e-3) < 1e-12
    with _pt.raises(AssertionError):
        error_bounded_ties([0, 1, 2], got, want, 3)          # not the top-k of its own scores
    bad = want.copy()
    bad[4] = 3.5                                             # index 4 displaces 2: error 2.5, but band is 5
    assert error_bounded_ties([0, 1, 4], bad, want, 3)[0] == 2
    bad2 = want.copy()
    bad2[2], bad2[3] = 2.0, 3.2                              # eps 1.0, band 2.0: 3 vs 2 differ by 1e-3, allowed
    assert error_bounded_ties([0, 1, 3], bad2, want, 3)[0] == 2
