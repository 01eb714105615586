"""GPU parity: every kernel of the path called through the C ABI against the oracle on the same inputs.

Bars: score / select / gather / origin bit-exact (no near-tie band is needed — the device reproduces
the reference's sequential double sums); attention |o - o_ref| <= 1e-2 + 1e-2 |o_ref| (bf16 output) against the
double restatement and a torch fp32 reference; SnapKV scores rel 1e-4 (fp32 math) with index sets bit-exact unless
the oracle's boundary gap is within the stated near-tie band.
"""
import hashlib
import os
import math
from pathlib import Path

import numpy as np
import pytest
import torch

import paper_2505_16175_b200 as qp
from oracle import oracle as O
from tiecheck import error_bounded_ties

pytestmark = pytest.mark.gpu
GOLD = __import__("pathlib").Path(__file__).resolve().parent / "golden"


def bf16_bits(t: torch.Tensor) -> np.ndarray:
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def f32_of(t: torch.Tensor) -> np.ndarray:
    return t.float().cpu().numpy()


def synth_groups(sizes, heads, width, tag, head_scale, device, seed=1):
    parts = [qp.synth_bf16(seed, tag, 0, g, n, heads, width, head_scale, device) for g, n in enumerate(sizes)]
    return torch.cat(parts, 0).contiguous()


# ------------------------------------------------------------------------------------------------ synth
def test_device_synth_matches_host(cuda):
    d = qp.synth_bf16(1, 1, 0, 3, 300, 4, 128, True, cuda)
    h = O.synth_bf16(1, 1, 0, 3, 300, 4, 128, True)
    assert bf16_bits(d).tobytes() == h.tobytes()


# ------------------------------------------------------------------------------------------------ scores
@pytest.mark.parametrize("sizes,heads,width", [([256] * 4, 2, 64), ([4096, 100, 1, 777], 4, 128), ([300], 1, 512)])
def test_norm_scores_bitexact_bf16(cuda, sizes, heads, width):
    plan = qp.GroupPlan.from_sizes(sizes, 0.5)
    g = plan.to(cuda)
    k = synth_groups(sizes, heads, width, 1, True, cuda)
    v = synth_groups(sizes, heads, width, 2, False, cuda)
    for scorer, x, neg in ((qp.Scorer.key_norm_small, k, True), (qp.Scorer.value_norm, v, False)):
        got = qp.score(k, v, g, heads, width, scorer).cpu().numpy()
        xf = f32_of(x)
        for gi, n in enumerate(sizes):
            t0 = plan.tok_off[gi]
            want = O.score_norm(xf[t0:t0 + n], heads, width, neg).ravel()
            seg = got[heads * t0: heads * (t0 + n)]
            assert seg.tobytes() == want.tobytes(), (scorer, gi)


def test_norm_scores_bitexact_bf16_extremes(cuda):
    """Arbitrary finite bf16 bit patterns (subnormals, zeros, +-huge, mixed scales): still bit-identical."""
    rng = np.random.default_rng(7)
    sizes, heads, width = [513, 64], 4, 128
    bits = rng.integers(0, 1 << 16, (sum(sizes), heads, width), dtype=np.uint32).astype(np.uint16)
    bits[(bits & 0x7f80) == 0x7f80] &= 0xbfff  # no inf/nan
    bits[:, 1, :] = 0  # all-zero rows -> -0.0
    bits[5, 2, :] = 0x0001  # all-subnormal row
    x = torch.from_numpy(bits.view(np.int16)).view(torch.bfloat16).to(cuda)
    plan = qp.GroupPlan.from_sizes(sizes, 0.5)
    g = plan.to(cuda)
    got = qp.score(x, x, g, heads, width, qp.Scorer.key_norm_small).cpu().numpy()
    xf = f32_of(x)
    for gi, n in enumerate(sizes):
        t0 = plan.tok_off[gi]
        want = O.score_norm(xf[t0:t0 + n], heads, width, True).ravel()
        assert got[heads * t0: heads * (t0 + n)].tobytes() == want.tobytes(), gi


@pytest.mark.parametrize("n,n_h,d_h", [(64, 4, 16), (257, 2, 64), (33, 1, 3)])
def test_reference_scores_f32_bitexact(cuda, n, n_h, d_h):
    rng = np.random.default_rng(n)
    k = (rng.standard_normal(n * n_h * d_h) * np.exp(rng.standard_normal(n * n_h * d_h))).astype(np.float32)
    v = rng.standard_normal(n * n_h * d_h).astype(np.float32)
    q = rng.standard_normal(5 * n_h * d_h).astype(np.float32)
    for scorer in (qp.Scorer.key_norm_small, qp.Scorer.value_norm, qp.Scorer.attention_score):
        got = qp.score_tokens(k, v, n, n_h, d_h, scorer, q)
        if O.ref is not None:
            want = O.ref_score_tokens(k, v, n, n_h, d_h, int(scorer), q)
        elif scorer == qp.Scorer.attention_score:
            want = O.score_attention(k, n, n_h, d_h, q, 5)
        else:
            want = O.score_norm(k if scorer == 0 else v, 1, n_h * d_h, scorer == 0)[0]
        assert got.tobytes() == want.tobytes(), scorer


# ------------------------------------------------------------------------------------------------ select
@pytest.mark.parametrize("sizes", [[1], [2, 3, 5], [256] * 4, [4096, 4095, 17], [16384], [30000]])
@pytest.mark.parametrize("kind", ["normal", "ties", "signed_zero", "constant"])
def test_select_matches_oracle(cuda, sizes, kind):
    rng = np.random.default_rng(sum(sizes))
    heads = 2
    segs = []
    for n in sizes:
        for _h in range(heads):
            if kind == "normal":
                s = rng.standard_normal(n)
            elif kind == "ties":
                s = rng.integers(-4, 5, n).astype(np.float64) * 0.5
            elif kind == "signed_zero":
                s = np.where(rng.random(n) < 0.5, -0.0, 0.0)
                s[rng.random(n) < 0.1] = 1.0
            else:
                s = np.full(n, -3.25)
            segs.append(s)
    for rho in (0.125, 0.5, 0.999):
        plan = qp.GroupPlan.from_sizes(sizes, rho)
        g = plan.to(cuda)
        got = qp.select(torch.from_numpy(np.concatenate(segs)).to(cuda), g, heads).cpu().numpy()
        for gi, n in enumerate(sizes):
            kk = plan.keep[gi]
            for h in range(heads):
                want = O.top_k(segs[gi * heads + h], kk)
                rows = got[(plan.row_off[gi]) * heads: (plan.row_off[gi] + kk) * heads].reshape(kk, heads)[:, h]
                assert rows.tolist() == want.tolist(), (gi, h, rho)


def test_top_k_indices_mirror(cuda):
    assert qp.top_k_indices(np.array([1, 3, 2, 3.0]), 2).tolist() == [1, 3]
    assert qp.top_k_indices(np.array([-0.0, 0.0, -0.0, 0.0]), 2).tolist() == [0, 1]
    assert qp.top_k_indices(np.array([1.0, 2.0]), 0).tolist() == []
    assert qp.top_k_indices(np.array([1.0, 2.0]), 5).tolist() == [0, 1]


# ------------------------------------------------------------------------------------------------ gather / prune
def test_golden_gqa_prune(cuda):
    """C1 GQA variant: per-head pruning on the device == the reference's per-head-slice prune_group fixture."""
    z = np.load(GOLD / "c1_gqa.npz")
    G, N, H, D, rho = int(z["G"]), int(z["N"]), int(z["H"]), int(z["D"]), float(z["rho"])
    plan = qp.GroupPlan.from_sizes([N] * G, rho)
    g = plan.to(cuda)
    k = synth_groups([N] * G, H, D, 1, True, cuda)
    v = synth_groups([N] * G, H, D, 2, False, cuda)
    kc, vc, origin, idx = qp.prune(k, v, g, H, D, qp.Scorer.key_norm_small, rho)
    kk = plan.keep[0]
    idx = idx.cpu().numpy().reshape(-1, H)
    kcf = f32_of(kc.view(-1, H, D))
    vcf = f32_of(vc.view(-1, H, D))
    org = origin.cpu().numpy().reshape(-1, H)
    for gi in range(G):
        r0 = plan.row_off[gi]
        for h in range(H):
            want = z[f"g{gi}_h{h}_idx"]
            assert idx[r0:r0 + kk, h].tolist() == want.tolist()
            assert org[r0:r0 + kk, h].tolist() == (plan.tok_off[gi] + want.astype(np.int64)).tolist()
            assert hashlib.sha256(np.ascontiguousarray(kcf[r0:r0 + kk, h]).tobytes()).digest() == bytes(
                z[f"g{gi}_h{h}_k_sha"])
            assert hashlib.sha256(np.ascontiguousarray(vcf[r0:r0 + kk, h]).tobytes()).digest() == bytes(
                z[f"g{gi}_h{h}_v_sha"])


@pytest.mark.parametrize("rho", [0.125, 0.25, 0.5, 1.0])
def test_prune_group_mirror_vs_reference(cuda, rho):
    n, n_h, d_h = 300, 4, 16
    rng = np.random.default_rng(int(rho * 1000))
    k = rng.integers(-3, 4, n * n_h * d_h).astype(np.float32)  # many exact score ties
    v = rng.standard_normal(n * n_h * d_h).astype(np.float32)
    q = rng.standard_normal(7 * n_h * d_h).astype(np.float32)
    for scorer in (qp.Scorer.key_norm_small, qp.Scorer.value_norm, qp.Scorer.attention_score):
        got = qp.prune_group(k, v, n, n_h, d_h, qp.PruneConfig(scorer, rho), q)
        if O.ref is None:
            continue
        kr, vr, ir = O.ref_prune_group(k, v, n, n_h, d_h, int(scorer), rho, q)
        assert got.indices.tolist() == ir.tolist()
        assert got.k.tobytes() == kr.tobytes() and got.v.tobytes() == vr.tobytes()


def test_prune_properties_full_c2(cuda):
    """BASELINE configs[1] sizes: 16 groups x 4096 tokens, 4 KV heads x 128: sortedness, counts, origins, copies,
    monotone inclusion I(rho1) subset I(rho2)."""
    sizes = [4096] * 16
    H, D = 4, 128
    k = synth_groups(sizes, H, D, 1, True, cuda)
    v = synth_groups(sizes, H, D, 2, False, cuda)
    sets = {}
    for rho in (0.125, 0.25, 0.5):
        plan = qp.GroupPlan.from_sizes(sizes, rho)
        g = plan.to(cuda)
        kc, vc, origin, idx = qp.prune(k, v, g, H, D, qp.Scorer.key_norm_small, rho)
        ix = idx.view(-1, H).cpu().numpy().astype(np.int64)
        kk = plan.keep[0]
        assert kk == qp.retained_count(rho, 4096)
        seg = ix.reshape(16, kk, H)
        assert (np.diff(seg, axis=1) > 0).all()  # strictly ascending per (group, head)
        src = (torch.from_numpy(seg).to(cuda) + torch.from_numpy(plan.tok_off[:-1]).to(cuda)[:, None, None])
        heads = torch.arange(H, device=cuda)[None, None, :]
        assert torch.equal(k[src.view(-1, H), heads.view(1, H)].reshape(-1), kc.view(-1))
        assert torch.equal(v[src.view(-1, H), heads.view(1, H)].reshape(-1), vc.view(-1))
        assert torch.equal(origin.view(-1, H), src.view(-1, H))
        sets[rho] = seg
    for a, b in ((0.125, 0.25), (0.25, 0.5)):
        for gi in range(16):
            for h in range(H):
                assert set(sets[a][gi, :, h].tolist()) <= set(sets[b][gi, :, h].tolist())
    # exact oracle check on two sampled groups
    plan = qp.GroupPlan.from_sizes(sizes, 0.5)
    kf = f32_of(k)
    for gi in (0, 11):
        t0 = plan.tok_off[gi]
        want = O.select_heads(O.score_norm(kf[t0:t0 + 4096], H, D, True), 4096, H, plan.keep[gi])
        assert (sets[0.5][gi] == want).all()


@pytest.mark.parametrize("n", [65536, 70001])
def test_prune_maximum_group_sizes_vs_oracle(cuda, n):
    """The largest group the fused kernel takes (16 CTAs x 4096 rows = 65536 tokens) and one past it (the three
    separate kernels take over), per KV head, against the oracle's exact select."""
    H, D, rho = 2, 64, 0.25
    plan = qp.GroupPlan.from_sizes([n], rho)
    g = plan.to(cuda)
    k = synth_groups([n], H, D, 5, True, cuda)
    v = synth_groups([n], H, D, 6, False, cuda)
    kc, vc, origin, idx = qp.prune(k, v, g, H, D, qp.Scorer.key_norm_small, rho)
    kk = plan.keep[0]
    want = O.select_heads(O.score_norm(f32_of(k), H, D, True), n, H, kk).astype(np.int64)
    got = idx.view(-1, H).cpu().numpy().astype(np.int64)
    assert (got == want).all()
    src = torch.from_numpy(want).to(cuda)
    heads = torch.arange(H, device=cuda)[None, :]
    assert torch.equal(k[src, heads].reshape(-1), kc.view(-1))
    assert torch.equal(v[src, heads].reshape(-1), vc.view(-1))


def test_identity_rho_one(cuda):
    sizes = [100, 37]
    plan = qp.GroupPlan.from_sizes(sizes, 1.0)
    g = plan.to(cuda)
    k = synth_groups(sizes, 2, 64, 1, True, cuda)
    v = synth_groups(sizes, 2, 64, 2, False, cuda)
    kc, vc, origin, idx = qp.prune(k, v, g, 2, 64, qp.Scorer.key_norm_small, 1.0)
    assert qp.last_prune_route() == 2
    assert torch.equal(kc.view_as(k), k) and torch.equal(vc.view_as(v), v)
    assert origin.view(-1, 2)[:, 0].tolist() == list(range(137))
    # the identity path fills idx like every scored path: 0..keep-1 per group and head
    want = torch.cat([torch.arange(n, device=cuda) for n in sizes]).view(-1, 1).expand(-1, 2)
    assert torch.equal(idx.view(-1, 2).long(), want)


# ------------------------------------------------------------------------------------------------ attention
def torch_attention(q, k, v, sizes, n_q, n_kv, scale):
    """Plain PyTorch fp32 causal GQA attention per group (reference for the tcgen05 kernel)."""
    outs, t0 = [], 0
    for n in sizes:
        qs = q[t0:t0 + n].float().permute(1, 0, 2)
        ks = k[t0:t0 + n].float().permute(1, 0, 2).repeat_interleave(n_q // n_kv, 0)
        vs = v[t0:t0 + n].float().permute(1, 0, 2).repeat_interleave(n_q // n_kv, 0)
        s = (qs @ ks.transpose(1, 2)) * scale
        s = s.masked_fill(torch.triu(torch.ones(n, n, dtype=torch.bool, device=q.device), 1), float("-inf"))
        outs.append((torch.softmax(s, -1) @ vs).permute(1, 0, 2))
        t0 += n
    return torch.cat(outs, 0)


def check_tol(got, want, what):
    err = (got.float() - want.float()).abs()
    bound = 1e-2 + 1e-2 * want.float().abs()
    bad = (err > bound).sum().item()
    assert bad == 0, f"{what}: {bad} elements out of tolerance; max abs err {err.max().item():.3e}"
    return err.max().item()


@pytest.mark.parametrize("sizes,n_q,n_kv,d", [([128], 1, 1, 128), ([256], 2, 1, 128), ([384, 100, 1, 129], 28, 4, 128),
                                              ([4096], 28, 4, 128), ([4096] * 2 + [1000], 28, 4, 128),
                                              ([16384], 4, 4, 128), ([256] * 4, 4, 2, 64), ([1000, 37, 4096], 28, 4, 64),
                                              # 320 ragged groups: the unit order's group blocks (~32 MB of K/V
                                              # each) give 6 blocks, the last one short
                                              ([128, 300, 17, 256] * 80, 28, 4, 128)])
def test_attention_vs_torch_fp32(cuda, sizes, n_q, n_kv, d):
    plan = qp.GroupPlan.from_sizes(sizes, 0.5)
    g = plan.to(cuda)
    q = synth_groups(sizes, n_q, d, 3, False, cuda)
    k = synth_groups(sizes, n_kv, d, 1, True, cuda)
    v = synth_groups(sizes, n_kv, d, 2, False, cuda)
    o = qp.attention(q, k, v, g, n_q, n_kv)
    torch.cuda.synchronize()
    want = torch_attention(q, k, v, sizes, n_q, n_kv, 1 / math.sqrt(d))
    check_tol(o, want, f"attention {sizes} d={d}")


@pytest.mark.parametrize("sizes,n_q,n_kv", [([256], 2, 1), ([384, 100, 1, 129], 28, 4), ([4096, 1000], 28, 4),
                                            ([255, 257, 513], 8, 2)])
def test_attention_cta_pair_variant_vs_torch_fp32(cuda, sizes, n_q, n_kv):
    """The experimental CTA-pair attention (attention2.cu, QVK_ATTN_2CTA=1: M = 256 pair MMAs, double-buffered S,
    column-split softmax) against torch fp32 — ragged groups, 1-token groups, long groups with lazy O rescales."""
    q = synth_groups(sizes, n_q, 128, 3, False, cuda)
    k = synth_groups(sizes, n_kv, 128, 1, True, cuda)
    v = synth_groups(sizes, n_kv, 128, 2, False, cuda)
    g = qp.GroupPlan.from_sizes(sizes, 0.5).to(cuda)
    os.environ["QVK_ATTN_2CTA"] = "1"
    try:
        o = qp.attention(q, k, v, g, n_q, n_kv)
        torch.cuda.synchronize()
    finally:
        del os.environ["QVK_ATTN_2CTA"]
    check_tol(o, torch_attention(q, k, v, sizes, n_q, n_kv, 1 / math.sqrt(128)), "cta-pair attention")


def test_attention_one_step_units_no_deadlock(cuda):
    """C3 shape (1024-token groups): thousands of 1-step head-pair units per launch.  The softmax warps must not run
    two units ahead of the epilogue (mbarrier phase aliasing deadlocked this shape once)."""
    sizes, n_q, n_kv = [1024] * 40, 28, 4
    plan = qp.GroupPlan.from_sizes(sizes, 0.25)
    g = plan.to(cuda)
    q = synth_groups(sizes, n_q, 128, 3, False, cuda)
    k = synth_groups(sizes, n_kv, 128, 1, True, cuda)
    v = synth_groups(sizes, n_kv, 128, 2, False, cuda)
    for _ in range(3):
        o = qp.attention(q, k, v, g, n_q, n_kv)
    torch.cuda.synchronize()
    check_tol(o[:4096], torch_attention(q[:4096], k[:4096], v[:4096], sizes[:4], n_q, n_kv, 1 / math.sqrt(128)),
              "1-step units")


def test_attention_persistent_many_units(cuda):
    """More work units than SMs with ragged groups: every CTA runs several units back to back (TMEM / barrier
    phases carried across units), including units whose second query tile is absent."""
    sizes, n_q, n_kv = [1100, 129, 4096, 300, 2000, 77], 28, 4
    plan = qp.GroupPlan.from_sizes(sizes, 0.5)
    g = plan.to(cuda)
    q = synth_groups(sizes, n_q, 128, 3, False, cuda)
    k = synth_groups(sizes, n_kv, 128, 1, True, cuda)
    v = synth_groups(sizes, n_kv, 128, 2, False, cuda)
    o1 = qp.attention(q, k, v, g, n_q, n_kv)
    o2 = qp.attention(q, k, v, g, n_q, n_kv)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2), "attention must be deterministic"
    check_tol(o1, torch_attention(q, k, v, sizes, n_q, n_kv, 1 / math.sqrt(128)), "persistent")


def test_attention_vs_double_oracle(cuda):
    sizes, n_q, n_kv = [300, 129], 28, 4
    plan = qp.GroupPlan.from_sizes(sizes, 0.5)
    g = plan.to(cuda)
    q = synth_groups(sizes, n_q, 128, 3, False, cuda)
    k = synth_groups(sizes, n_kv, 128, 1, True, cuda)
    v = synth_groups(sizes, n_kv, 128, 2, False, cuda)
    o = qp.attention(q, k, v, g, n_q, n_kv)
    t0 = 0
    for n in sizes:
        want = O.attention(f32_of(q[t0:t0 + n]), f32_of(k[t0:t0 + n]), f32_of(v[t0:t0 + n]), n_q, n_kv, 128,
                           1 / math.sqrt(128))
        check_tol(o[t0:t0 + n], torch.from_numpy(want).to(cuda), f"group of {n}")
        t0 += n


# ------------------------------------------------------------------------------------------------ SnapKV
@pytest.mark.parametrize("sizes,window,pool,n_q,n_kv", [
    ([256, 100], 32, 1, 28, 4), ([1024], 32, 7, 28, 4), ([20], 32, 1, 28, 4),
    # gq * W > 256: the window rows are cut into blocks of <= 256 operand rows run one after another
    ([300, 1024], 64, 1, 28, 4),   # 2 blocks of 32 window rows (224 operand rows each)
    ([700, 129], 50, 3, 28, 4),    # 2 blocks of 25 rows, pooled
    ([40, 513], 64, 1, 28, 4),     # window longer than the first group (rows before the group masked)
    ([600], 100, 1, 16, 2),        # gq 8: 4 blocks of 25 rows
    ([333], 300, 1, 4, 4),         # gq 1, W 300 > 256: 2 blocks of 150 rows
])
def test_snapkv_vs_oracle(cuda, sizes, window, pool, n_q, n_kv):
    plan = qp.GroupPlan.from_sizes(sizes, 0.25)
    g = plan.to(cuda)
    q = synth_groups(sizes, n_q, 128, 3, False, cuda)
    k = synth_groups(sizes, n_kv, 128, 1, True, cuda)
    got = qp.snapkv_scores(q, k, g, n_q, n_kv, window, pool).cpu().numpy()
    t0 = 0
    for gi, n in enumerate(sizes):
        want = O.snapkv_scores(f32_of(q[t0:t0 + n]), f32_of(k[t0:t0 + n]), n_q, n_kv, 128, window, pool,
                               1 / math.sqrt(128))
        seg = got[n_kv * t0: n_kv * (t0 + n)].reshape(n_kv, n)
        np.testing.assert_allclose(seg, want, rtol=1e-4, atol=1e-6)
        # index sets, barring near-ties: an index may be in one set and not the other only if its oracle score lies
        # within tau = 1e-4 (relative, the fp32 scores' tolerance) of the oracle's k-th score; the count is reported
        kk = plan.keep[gi]
        for h in range(n_kv):
            got_set = set(O.top_k(seg[h], kk).tolist())
            order = np.argsort(-want[h], kind="stable")
            want_set = set(order[:kk].tolist())
            kth = want[h][order[kk - 1]]
            diff = got_set ^ want_set
            near = [i for i in diff if abs(want[h][i] - kth) <= 1e-4 * abs(kth)]
            assert len(diff) == len(near), f"group {gi} head {h}: index differences outside the near-tie band"
            # and the tighter, error-derived band: differences only within 2 x this head's measured score error
            nd, eps, band = error_bounded_ties(sorted(got_set), seg[h], want[h], kk)
            print(f"snapkv group {gi} head {h}: {nd} near-tie index differences, eps {eps:.3g} "
                  f"(rel {eps / max(abs(kth), 1e-300):.3g} of the k-th score)")
        t0 += n


# ------------------------------------------------------------------------------------------------ full layer
@pytest.mark.parametrize("scorer,per_head", [(qp.Scorer.key_norm_small, True), (qp.Scorer.value_norm, False)])
def test_prefill_layer(cuda, scorer, per_head):
    sizes, n_q, n_kv, D, rho = [1024, 1024, 512], 28, 4, 128, 0.25
    plan = qp.GroupPlan.from_sizes(sizes, rho)
    g = plan.to(cuda)
    q = synth_groups(sizes, n_q, D, 3, False, cuda)
    k = synth_groups(sizes, n_kv, D, 1, True, cuda)
    v = synth_groups(sizes, n_kv, D, 2, False, cuda)
    buf = qp.prefill_layer(q, k, v, g, n_q, n_kv, rho, scorer, per_head)
    torch.cuda.synchronize()
    check_tol(buf.o, torch_attention(q, k, v, sizes, n_q, n_kv, 1 / math.sqrt(D)), "layer attention")
    heads, width = (n_kv, D) if per_head else (1, n_kv * D)
    sc = qp.score(k, v, g, heads, width, scorer)
    idx = qp.select(sc, g, heads)
    kc, vc, origin = qp.gather(k, v, g, heads, width, idx)
    assert torch.equal(buf.idx[: idx.numel()], idx)
    assert torch.equal(buf.k_cache, kc) and torch.equal(buf.v_cache, vc) and torch.equal(buf.origin, origin)


@pytest.mark.parametrize("sizes,window,pool,n_q,n_kv", [
    ([1024, 1024, 512], 32, 1, 28, 4),
    ([700, 20, 1300], 64, 3, 28, 4),   # 2 window blocks, a group shorter than the window, pooling
    ([600, 129], 100, 1, 16, 2),       # GQA 8, 4 blocks
])
def test_prefill_layer_snapkv_window_stats_from_attention(cuda, sizes, window, pool, n_q, n_kv):
    """qvk_prefill_layer with SnapKV: pass 1 (the window rows' softmax statistics) comes out of the layer's attention
    kernel and the scorer runs pass 2 only.  Scores within rel 1e-4 of the fp64 restatement, index sets equal barring
    near-ties (same band as the standalone scorer), cache = the indexed K/V rows."""
    D, rho = 128, 0.25
    plan = qp.GroupPlan.from_sizes(sizes, rho)
    g = plan.to(cuda)
    q = synth_groups(sizes, n_q, D, 3, False, cuda)
    k = synth_groups(sizes, n_kv, D, 1, True, cuda)
    v = synth_groups(sizes, n_kv, D, 2, False, cuda)
    buf = qp.prefill_layer(q, k, v, g, n_q, n_kv, rho, qp.Scorer.snapkv, True, snap_window=window, snap_pool=pool)
    torch.cuda.synchronize()
    check_tol(buf.o, torch_attention(q, k, v, sizes, n_q, n_kv, 1 / math.sqrt(D)), "layer attention")
    kc, vc, origin = qp.gather(k, v, g, n_kv, D, buf.idx)
    assert torch.equal(buf.k_cache, kc) and torch.equal(buf.v_cache, vc) and torch.equal(buf.origin, origin)
    got = buf.scores.cpu().numpy()
    standalone = qp.snapkv_scores(q, k, g, n_q, n_kv, window, pool).cpu().numpy()
    np.testing.assert_allclose(got, standalone, rtol=1e-4, atol=1e-6)
    t0 = 0
    for gi, n in enumerate(sizes):
        want = O.snapkv_scores(f32_of(q[t0:t0 + n]), f32_of(k[t0:t0 + n]), n_q, n_kv, D, window, pool,
                               1 / math.sqrt(D))
        seg = got[n_kv * t0: n_kv * (t0 + n)].reshape(n_kv, n)
        np.testing.assert_allclose(seg, want, rtol=1e-4, atol=1e-6)
        kk, r0 = int(plan.keep[gi]), int(plan.row_off[gi])
        idx = buf.idx[r0 * n_kv:(r0 + kk) * n_kv].view(kk, n_kv).cpu().numpy()
        for h in range(n_kv):
            order = np.argsort(-want[h], kind="stable")
            kth = want[h][order[kk - 1]]
            diff = set(order[:kk].tolist()) ^ set(idx[:, h].tolist())
            near = [i for i in diff if abs(want[h][i] - kth) <= 1e-4 * abs(kth)]
            assert len(diff) == len(near), f"group {gi} head {h}: index differences outside the near-tie band"
        t0 += n


@pytest.mark.parametrize("sizes,window,n_q,n_kv", [([700, 20, 1300], 64, 28, 4), ([256, 129], 32, 8, 2)])
def test_attention_window_stats_and_snapkv_pass2(cuda, sizes, window, n_q, n_kv):
    """qvk_attention_window_stats: the softmax statistics of each group's last `window` rows equal
    log2(sum_j exp(scale q.k_j)) (fp64 from the bf16 inputs) within 2e-4 (log2 units); the output is the plain
    attention's bit for bit; qvk_snapkv_score_stats on them matches the oracle like the two-pass scorer."""
    D = 128
    scale = 1 / math.sqrt(D)
    plan = qp.GroupPlan.from_sizes(sizes, 0.25)
    g = plan.to(cuda)
    q = synth_groups(sizes, n_q, D, 3, False, cuda)
    k = synth_groups(sizes, n_kv, D, 1, True, cuda)
    v = synth_groups(sizes, n_kv, D, 2, False, cuda)
    o, st = qp.attention_window_stats(q, k, v, g, n_q, n_kv, window)
    assert torch.equal(o, qp.attention(q, k, v, g, n_q, n_kv))
    t0 = 0
    for gi, n in enumerate(sizes):
        qd, kd = q[t0:t0 + n].double(), k[t0:t0 + n].double()
        for r in range(max(0, window - n), window):
            pos = n - window + r
            for h in range(n_q):
                x = (kd[:pos + 1, h // (n_q // n_kv)] @ qd[pos, h]) * scale
                want = torch.logsumexp(x, 0).item() / math.log(2)
                got = st[gi, h, r].item()
                assert abs(got - want) <= 2e-4, (gi, r, h, got, want)
        t0 += n
    got = qp.snapkv_scores(q, k, g, n_q, n_kv, window, window_stats=st).cpu().numpy()
    t0 = 0
    for gi, n in enumerate(sizes):
        want = O.snapkv_scores(f32_of(q[t0:t0 + n]), f32_of(k[t0:t0 + n]), n_q, n_kv, D, window, 1, scale)
        np.testing.assert_allclose(got[n_kv * t0: n_kv * (t0 + n)].reshape(n_kv, n), want, rtol=1e-4, atol=1e-6)
        t0 += n


def test_host_prefill_pipeline_matches_device_layer(cuda):
    """Chunked host-buffer pipeline (copies overlapped with kernels) == one device-resident prefill_layer call."""
    sizes, n_q, n_kv, rho = [1024, 1024, 1024, 777, 1024], 28, 4, 0.5
    plan = qp.GroupPlan.from_sizes(sizes, rho)
    g = plan.to(cuda)
    q = synth_groups(sizes, n_q, 128, 3, False, cuda)
    k = synth_groups(sizes, n_kv, 128, 1, True, cuda)
    v = synth_groups(sizes, n_kv, 128, 2, False, cuda)
    buf = qp.prefill_layer(q, k, v, g, n_q, n_kv, rho)
    hp = qp.HostPrefill(plan, n_q, n_kv, 128, rho, cuda, chunks=3)
    hq, hk, hv = (t.cpu().pin_memory() for t in (q, k, v))
    out_k = torch.empty(hp.k_cache.numel(), dtype=torch.bfloat16).pin_memory()
    out_v = torch.empty_like(out_k).pin_memory()
    out_o = torch.empty(hp.origin.numel(), dtype=torch.int64).pin_memory()
    for _ in range(2):
        hp.run(hq, hk, hv, out_k, out_v, out_o)
    torch.cuda.synchronize()
    assert torch.equal(out_k, buf.k_cache.cpu()) and torch.equal(out_v, buf.v_cache.cpu())
    assert torch.equal(out_o, buf.origin.cpu())
    assert torch.equal(hp.o, buf.o)


# ------------------------------------------------------------------------------------------------ fused prune
def _separate_prune(k, v, g, heads, width, scorer):
    """score -> select -> gather as three launches (score.cu, select.cu, gather.cu): the fused kernel's check."""
    sc = qp.score(k, v, g, heads, width, scorer)
    idx = qp.select(sc, g, heads)
    kc, vc, origin = qp.gather(k, v, g, heads, width, idx)
    return sc, idx, kc, vc, origin


def _tie_rows(sizes, heads, width, device, seed):
    """Integer-valued bf16 rows from {-1, 0, 1}: norms collide massively (exact ties straddle every k boundary);
    some rows all-zero (score -0.0 == +0.0)."""
    gen = torch.Generator().manual_seed(seed)
    x = torch.randint(-1, 2, (sum(sizes), heads, width), generator=gen).float()
    x[::7] = 0.0
    return x.to(torch.bfloat16).to(device)


@pytest.mark.parametrize("sizes,heads,width,rho,kind", [
    ([4096] * 3, 4, 128, 0.5, "synth"),
    ([4096, 100, 1, 777, 3, 16384, 2], 4, 128, 0.25, "synth"),
    ([256] * 4, 2, 64, 0.5, "synth"),
    ([300, 5, 1000], 1, 512, 0.5, "synth"),
    ([1000, 999, 8], 2, 256, 0.125, "synth"),
    ([2048, 513, 64], 4, 128, 0.5, "ties"),
    ([777, 31], 1, 512, 0.25, "ties"),
    ([1500, 40000], 2, 64, 0.3, "synth"),
])
def test_prune_fused_matches_separate_kernels(cuda, sizes, heads, width, rho, kind):
    """qvk_prune's one-launch cluster kernel (prune_fused.cu) == the three separate kernels, bit for bit: scores,
    retained indices, cache rows, origins — ragged groups, 1-token groups (k == N), massive exact ties."""
    plan = qp.GroupPlan.from_sizes(sizes, rho)
    g = plan.to(cuda)
    if kind == "ties":
        k, v = _tie_rows(sizes, heads, width, cuda, 1), _tie_rows(sizes, heads, width, cuda, 2)
    else:
        k = synth_groups(sizes, heads, width, 1, True, cuda)
        v = synth_groups(sizes, heads, width, 2, False, cuda)
    for scorer in (qp.Scorer.key_norm_small, qp.Scorer.value_norm):
        kc, vc, origin, idx = qp.prune(k, v, g, heads, width, scorer, rho)
        sc, idx2, kc2, vc2, origin2 = _separate_prune(k, v, g, heads, width, scorer)
        torch.cuda.synchronize()
        R = plan.total_rows * heads
        assert torch.equal(idx[:R], idx2[:R]), scorer
        assert torch.equal(kc, kc2) and torch.equal(vc, vc2) and torch.equal(origin, origin2), scorer


@pytest.mark.parametrize("entry", ["prune", "prefill_layer"])
@pytest.mark.parametrize("scorer", [qp.Scorer.key_norm_small, qp.Scorer.value_norm])
def test_small_per_token_batches_route_to_separate_kernels(cuda, tmp_path, entry, scorer):
    """Default routing (QVK_PRUNE_FUSED_MIN_SEGS unset): a small per-token batch takes score + select + gather
    (qvk_last_prune_route() == 1) and yields the same cache as the fused kernel this test process is pinned to
    (route 0) — for qvk_prune and qvk_prefill_layer (per_head = 0), both norm scorers."""
    import subprocess
    import sys
    sizes, n_q, n_kv, d, rho = [300, 5, 1000], 8, 4, 128, 0.5
    code = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r); sys.path.insert(0, %r)
import paper_2505_16175_b200 as qp
from test_kernels_gpu import synth_groups
dev = torch.device('cuda', 0)
sizes, n_q, n_kv, d, rho, entry, scorer = %r, %d, %d, %d, %r, %r, qp.Scorer(%d)
plan = qp.GroupPlan.from_sizes(sizes, rho)
g = plan.to(dev)
k = synth_groups(sizes, n_kv, d, 1, True, dev); v = synth_groups(sizes, n_kv, d, 2, False, dev)
if entry == "prune":
    kc, vc, origin, idx = qp.prune(k.view(-1, 1, n_kv * d), v.view(-1, 1, n_kv * d), g, 1, n_kv * d, scorer, rho)
else:
    q = synth_groups(sizes, n_q, d, 3, False, dev)
    buf = qp.prefill_layer(q, k, v, g, n_q, n_kv, rho, scorer, False)
    kc, vc, origin = buf.k_cache, buf.v_cache, buf.origin
torch.cuda.synchronize()
print("route", qp.last_prune_route())
np.save(sys.argv[1], np.concatenate([kc.view(torch.int16).cpu().numpy().ravel().astype(np.int64),
                                     vc.view(torch.int16).cpu().numpy().ravel().astype(np.int64),
                                     origin.cpu().numpy().ravel()]))
""" % (str(Path(__file__).resolve().parent.parent), str(Path(__file__).resolve().parent), sizes, n_q, n_kv, d, rho,
       entry, int(scorer))
    outs = {}
    for mode, env_min in (("default", None), ("fused", "0")):
        env = {kk: vv for kk, vv in os.environ.items() if kk != "QVK_PRUNE_FUSED_MIN_SEGS"}
        if env_min is not None:
            env["QVK_PRUNE_FUSED_MIN_SEGS"] = env_min
        out = tmp_path / f"{mode}.npy"
        r = subprocess.run([sys.executable, "-c", code, str(out)], capture_output=True, text=True, env=env,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        route = int(r.stdout.split("route")[1].split()[0])
        assert route == (1 if mode == "default" else 0), (mode, route)
        outs[mode] = np.load(out)
    assert np.array_equal(outs["default"], outs["fused"])


def test_prune_fused_extreme_values(cuda):
    """Arbitrary finite bf16 bit patterns (subnormals, +-huge, mixed scales): the fused kernel's order-free sums
    take the sequential fallback where needed and still match the separate kernels bit for bit."""
    sizes, heads, width = [2000, 333], 4, 128
    gen = torch.Generator().manual_seed(7)
    bits = torch.randint(0, 0x7f80, (sum(sizes), heads, width), generator=gen, dtype=torch.int32)
    sign = torch.randint(0, 2, bits.shape, generator=gen, dtype=torch.int32) << 15
    k = (bits | sign).to(torch.int16).view(torch.bfloat16).to(cuda)
    v = synth_groups(sizes, heads, width, 2, False, cuda)
    plan = qp.GroupPlan.from_sizes(sizes, 0.5)
    g = plan.to(cuda)
    kc, vc, origin, idx = qp.prune(k, v, g, heads, width, qp.Scorer.key_norm_small, 0.5)
    sc, idx2, kc2, vc2, origin2 = _separate_prune(k, v, g, heads, width, qp.Scorer.key_norm_small)
    R = plan.total_rows * heads
    assert torch.equal(idx[:R], idx2[:R])
    assert torch.equal(kc, kc2) and torch.equal(origin, origin2)


def test_prune_fused_scores_zero_and_tiny_rows_bitexact(cuda):
    """The fused scoring's scaled conversion: zero elements enter as stand-ins that must vanish exactly, which needs
    every nonzero |x| >= 2^-90 (else the sequential fallback).  Rows mixing zeros with normal values, with values just
    above / below 2^-90, a lone tiny nonzero among zeros, all-zero rows and huge values: the fused kernel's double
    scores equal the separate key-norm kernel's bit for bit (both = the reference's sequential sums)."""
    heads, width, n = 4, 128, 1536
    gen = torch.Generator().manual_seed(11)
    x = torch.randn(n, heads, width, generator=gen)
    kind = torch.arange(n) % 8
    zero = torch.rand(n, heads, width, generator=gen) < 0.3
    x[(kind == 0)[:, None, None] & zero] = 0.0                                   # normal values, 30 % zeros
    x[kind == 1] = x[kind == 1] * 2.0 ** -89                                     # tiny, >= 2^-90 mostly
    x[(kind == 1)[:, None, None] & zero] = 0.0
    x[kind == 2] = x[kind == 2] * 2.0 ** -91                                     # below 2^-90: fallback
    x[(kind == 2)[:, None, None] & zero] = 0.0
    x[kind == 3] = 0.0                                                           # all zero
    x[kind == 4] = 0.0
    x[kind == 4, :, 5] = 2.0 ** -90                                              # lone tiny at the bound
    x[kind == 5] = x[kind == 5] * 2.0 ** 60                                      # huge
    x[(kind == 5)[:, None, None] & zero] = 0.0
    x[kind == 6] = 0.0
    x[kind == 6, :, ::17] = 1.0                                                  # sparse ones
    x[kind == 7] = x[kind == 7] * 2.0 ** -60                                     # small, zeros mixed
    x[(kind == 7)[:, None, None] & zero] = 0.0
    k = x.to(torch.bfloat16).to(cuda)
    v = synth_groups([n], heads, width, 2, False, cuda)
    plan = qp.GroupPlan.from_sizes([512, 1024], 0.5)
    g = plan.to(cuda)
    R = plan.total_rows
    sc = torch.empty(n * heads, dtype=torch.float64, device=cuda)
    idx = torch.empty(R * heads, dtype=torch.int32, device=cuda)
    kc = torch.empty(R * heads * width, dtype=torch.bfloat16, device=cuda)
    vc, org = torch.empty_like(kc), torch.empty(R * heads, dtype=torch.int64, device=cuda)
    s = torch.cuda.current_stream().cuda_stream
    for scorer in (qp.Scorer.key_norm_small, qp.Scorer.value_norm):
        x_in = (k, v) if scorer == qp.Scorer.key_norm_small else (v, k)
        qp._lib.check(qp.lib.qvk_prune(s, g.ref, x_in[0].data_ptr(), x_in[1].data_ptr(), qp._lib.QVK_BF16, heads,
                                       width, int(scorer), 0.5, None, 0, heads, sc.data_ptr(), idx.data_ptr(),
                                       kc.data_ptr(), vc.data_ptr(), org.data_ptr()))
        want = qp.score(x_in[0], x_in[1], g, heads, width, scorer)
        torch.cuda.synchronize()
        assert qp.last_prune_route() == 0, "the fused kernel must have run"
        assert torch.equal(sc.view(torch.int64), want.view(torch.int64)), scorer


@pytest.mark.parametrize("sizes,window", [([1024, 1024, 300], 32), ([4096, 77], 16)])
def test_select_gather_snapkv_matches_separate(cuda, sizes, window):
    """qvk_select_gather (one cluster launch from precomputed SnapKV scores) == qvk_select + qvk_gather."""
    n_q, n_kv, D, rho = 28, 4, 128, 0.25
    plan = qp.GroupPlan.from_sizes(sizes, rho)
    g = plan.to(cuda)
    q = synth_groups(sizes, n_q, D, 3, False, cuda)
    k = synth_groups(sizes, n_kv, D, 1, True, cuda)
    v = synth_groups(sizes, n_kv, D, 2, False, cuda)
    sc = qp.snapkv_scores(q, k, g, n_q, n_kv, window)
    kc, vc, origin, idx = qp.select_gather(sc, k, v, g, n_kv, D)
    idx2 = qp.select(sc, g, n_kv)
    kc2, vc2, origin2 = qp.gather(k, v, g, n_kv, D, idx2)
    R = plan.total_rows * n_kv
    assert torch.equal(idx[:R], idx2[:R])
    assert torch.equal(kc, kc2) and torch.equal(vc, vc2) and torch.equal(origin, origin2)


# ------------------------------------------------------------------------------------------------ projection (§8f-1)
def _proj_inputs(T, d_model, n_q, n_kv, d_h, device, seed=5):
    x = qp.synth_bf16(seed, 7, 0, 0, T, 1, d_model, False, device).view(T, d_model)
    w = (qp.synth_bf16(seed, 8, 0, 0, (n_q + 2 * n_kv) * d_h, 1, d_model, False, device).float()
         * (1.0 / math.sqrt(d_model))).to(torch.bfloat16).view(-1, d_model)
    return x, w


@pytest.mark.parametrize("sizes,d_model,n_q,n_kv,d_h", [([4096, 1000], 3584, 28, 4, 128), ([256] * 4, 256, 4, 2, 64),
                                                        ([77, 300], 512, 8, 4, 64), ([128], 1024, 4, 2, 128)])
def test_project_qkv_vs_torch_and_fused_keynorm(cuda, sizes, d_model, n_q, n_kv, d_h):
    """tcgen05 QKV GEMM vs a torch fp32 matmul of the same bf16 operands (|err| <= 1e-2 + 1e-2 |ref|: bf16 output
    rounding + accumulation order), and the key-norm fused into its epilogue == qvk_score on the stored K, bit for
    bit (prefill.cpp:200-212 order)."""
    T = sum(sizes)
    plan = qp.GroupPlan.from_sizes(sizes, 0.5)
    g = plan.to(cuda)
    x, w = _proj_inputs(T, d_model, n_q, n_kv, d_h, cuda)
    q, k, v, sc = qp.project_qkv(x, w, n_q, n_kv, d_h, g, with_scores=True)
    ref = x.float() @ w.float().t()
    qc, kc = n_q * d_h, n_kv * d_h
    check_tol(q.view(T, -1), ref[:, :qc], "Q")
    check_tol(k.view(T, -1), ref[:, qc:qc + kc], "K")
    check_tol(v.view(T, -1), ref[:, qc + kc:], "V")
    want = qp.score(k, v, g, n_kv, d_h, qp.Scorer.key_norm_small)
    assert sc.cpu().numpy().tobytes() == want.cpu().numpy().tobytes()


def test_prefill_layer_x_matches_projection_then_layer(cuda):
    """qvk_prefill_layer_x (projection with fused key-norm -> attention -> fused select/gather) == qvk_project_qkv
    followed by qvk_prefill_layer on its outputs, bit for bit."""
    sizes, d_model, n_q, n_kv, d_h, rho = [2048, 2048, 640], 3584, 28, 4, 128, 0.5
    T = sum(sizes)
    plan = qp.GroupPlan.from_sizes(sizes, rho)
    g = plan.to(cuda)
    x, w = _proj_inputs(T, d_model, n_q, n_kv, d_h, cuda, seed=9)
    buf, (q, k, v) = qp.prefill_layer_x(x, w, g, n_q, n_kv, d_h, rho)
    q2, k2, v2 = qp.project_qkv(x, w, n_q, n_kv, d_h)
    assert torch.equal(q, q2) and torch.equal(k, k2) and torch.equal(v, v2)
    buf2 = qp.prefill_layer(q2, k2, v2, g, n_q, n_kv, rho)
    torch.cuda.synchronize()
    R = plan.total_rows * n_kv
    assert torch.equal(buf.o, buf2.o)
    assert torch.equal(buf.idx[:R], buf2.idx[:R])
    assert torch.equal(buf.k_cache, buf2.k_cache) and torch.equal(buf.v_cache, buf2.v_cache)
    assert torch.equal(buf.origin, buf2.origin)


# ------------------------------------------------------------------------------------------------ decode consumer (§8f-4)
@pytest.mark.parametrize("n_tq,rows,n_q,n_kv", [(1, 32768, 28, 4), (3, 100, 28, 4), (64, 5000, 28, 4), (1, 1, 4, 2),
                                                (10, 70001, 8, 8), (40, 33333, 8, 2), (20, 129, 28, 4)])
def test_decode_attention_vs_torch(cuda, n_tq, rows, n_q, n_kv):
    """Query tokens attending over a pruned cache (non-causal, GQA) vs a torch fp32 reference: O within
    1e-2 + 1e-2 |ref| (bf16 output), natural-log LSE within 1e-3 absolute."""
    d = 128
    gen = torch.Generator(device=cuda).manual_seed(rows + n_tq)
    q = torch.randn(n_tq, n_q, d, device=cuda, generator=gen).to(torch.bfloat16)
    kc = torch.randn(rows, n_kv, d, device=cuda, generator=gen).to(torch.bfloat16)
    vc = torch.randn(rows, n_kv, d, device=cuda, generator=gen).to(torch.bfloat16)
    o, lse = qp.decode_attention(q, kc, vc, n_q, n_kv, with_lse=True)
    g = n_q // n_kv
    kf = kc.float().repeat_interleave(g, 1).permute(1, 0, 2)   # (n_q, rows, d)
    vf = vc.float().repeat_interleave(g, 1).permute(1, 0, 2)
    s = torch.einsum("thd,hrd->htr", q.float(), kf) / math.sqrt(d)
    ref = torch.einsum("htr,hrd->thd", torch.softmax(s, -1), vf)
    check_tol(o, ref, "decode O")
    lse_ref = torch.logsumexp(s, -1).t()
    assert (lse - lse_ref).abs().max().item() <= 1e-3


# ------------------------------------------------------------------------------------------------ frames -> pruned cache
def _frames(F, H, W, device, seed=3):
    gen = torch.Generator().manual_seed(seed)
    return torch.randint(0, 256, (F, 3, H, W), generator=gen, dtype=torch.uint8).to(device)


def test_tokenize_bf16_is_rounded_reference_tokens(cuda):
    """GPU stand-in tokenizer: the bf16 variant is exactly the fp32 reference tokens rounded to nearest even."""
    fr = _frames(4, 60, 64, cuda)  # tpf 48: 6 x 8 patch grid
    embed = ((torch.rand(256, 3, generator=torch.Generator().manual_seed(1)) * 2 - 1) / 255).to(cuda)
    t32 = qp.tokenize(fr, 48, embed)
    t16 = qp.tokenize(fr, 48, embed, bf16=True)
    assert torch.equal(t16, t32.to(torch.bfloat16))


def test_frame_prefill_matches_device_layer(cuda):
    """FramePrefill (host frames -> chunked upload, tokenize, projection, attention, prune, readback) == the same
    kernels on device-resident data in one call, bit for bit."""
    F, fpg, tpf, H, W = 24, 4, 64, 64, 64
    n_q, n_kv, d_h, d_model, rho = 8, 2, 128, 512, 0.5
    plan = qp.GroupPlan.plan(F, fpg, tpf, rho, 1)
    g = plan.to(cuda)
    fr = _frames(F, H, W, cuda)
    embed = ((torch.rand(d_model, 3, generator=torch.Generator().manual_seed(2)) * 2 - 1) / 255).to(cuda)
    w = (torch.randn((n_q + 2 * n_kv) * d_h, d_model, generator=torch.Generator().manual_seed(4)) /
         math.sqrt(d_model)).to(torch.bfloat16).to(cuda)
    x = qp.tokenize(fr, tpf, embed, bf16=True)
    buf, _ = qp.prefill_layer_x(x, w, g, n_q, n_kv, d_h, rho)
    fp = qp.FramePrefill(plan, tpf, H, W, embed, w, n_q, n_kv, d_h, rho, cuda, chunks=3)
    hf = fr.cpu().pin_memory()
    out_k = torch.empty(fp.k_cache.numel(), dtype=torch.bfloat16).pin_memory()
    out_v = torch.empty_like(out_k).pin_memory()
    out_o = torch.empty(fp.origin.numel(), dtype=torch.int64).pin_memory()
    for _ in range(2):
        fp.run(hf, out_k, out_v, out_o)
    torch.cuda.synchronize()
    assert torch.equal(out_k, buf.k_cache.cpu()) and torch.equal(out_v, buf.v_cache.cpu())
    assert torch.equal(out_o, buf.origin.cpu())
    assert torch.equal(fp.o, buf.o)


def test_frame_prefill_chained_calls(cuda):
    """run(join=False) chains consecutive calls (call i+1's uploads and kernels overlap call i's readback): three
    different videos back to back into three host output sets, each equal to its own device-path result."""
    F, fpg, tpf, H, W = 24, 4, 64, 64, 64
    n_q, n_kv, d_h, d_model, rho = 8, 2, 128, 512, 0.5
    plan = qp.GroupPlan.plan(F, fpg, tpf, rho, 1)
    g = plan.to(cuda)
    embed = ((torch.rand(d_model, 3, generator=torch.Generator().manual_seed(2)) * 2 - 1) / 255).to(cuda)
    w = (torch.randn((n_q + 2 * n_kv) * d_h, d_model, generator=torch.Generator().manual_seed(4)) /
         math.sqrt(d_model)).to(torch.bfloat16).to(cuda)
    fp = qp.FramePrefill(plan, tpf, H, W, embed, w, n_q, n_kv, d_h, rho, cuda, chunks=3)
    vids, outs, refs = [], [], []
    for seed in (31, 32, 33):
        fr = _frames(F, H, W, cuda, seed=seed)
        buf, _ = qp.prefill_layer_x(qp.tokenize(fr, tpf, embed, bf16=True), w, g, n_q, n_kv, d_h, rho)
        refs.append((buf.k_cache.cpu(), buf.v_cache.cpu(), buf.origin.cpu()))
        vids.append(fr.cpu().pin_memory())
        ok = torch.empty(fp.k_cache.numel(), dtype=torch.bfloat16).pin_memory()
        outs.append((ok, torch.empty_like(ok).pin_memory(),
                     torch.empty(fp.origin.numel(), dtype=torch.int64).pin_memory()))
    torch.cuda.synchronize()
    for hf, (ok, ov, oo) in zip(vids, outs):
        fp.run(hf, ok, ov, oo, join=False)
    fp.join()
    torch.cuda.synchronize()
    for (ok, ov, oo), (rk, rv, ro) in zip(outs, refs):
        assert torch.equal(ok, rk) and torch.equal(ov, rv) and torch.equal(oo, ro)


def test_frame_prefill_after_compute_hook(cuda):
    """after_compute (the multi-GPU all-gather in bench.py) runs on the caller's stream after the last chunk's
    kernels, sees the complete device cache, and the host outputs still receive every computed row."""
    F, fpg, tpf, H, W = 16, 4, 64, 64, 64
    n_q, n_kv, d_h, d_model, rho = 8, 2, 128, 512, 0.5
    plan = qp.GroupPlan.plan(F, fpg, tpf, rho, 1)
    g = plan.to(cuda)
    fr = _frames(F, H, W, cuda, seed=41)
    embed = ((torch.rand(d_model, 3, generator=torch.Generator().manual_seed(3)) * 2 - 1) / 255).to(cuda)
    w = (torch.randn((n_q + 2 * n_kv) * d_h, d_model, generator=torch.Generator().manual_seed(5)) /
         math.sqrt(d_model)).to(torch.bfloat16).to(cuda)
    buf, _ = qp.prefill_layer_x(qp.tokenize(fr, tpf, embed, bf16=True), w, g, n_q, n_kv, d_h, rho)
    fp = qp.FramePrefill(plan, tpf, H, W, embed, w, n_q, n_kv, d_h, rho, cuda, chunks=2)
    seen = torch.zeros_like(fp.k_cache)
    out_k = torch.empty(fp.k_cache.numel(), dtype=torch.bfloat16).pin_memory()
    out_v = torch.empty_like(out_k).pin_memory()
    out_o = torch.empty(fp.origin.numel(), dtype=torch.int64).pin_memory()
    fp.run(fr.cpu().pin_memory(), out_k, out_v, out_o, after_compute=lambda: seen.copy_(fp.k_cache))
    torch.cuda.synchronize()
    assert torch.equal(seen.view(-1).cpu(), buf.k_cache.cpu())
    assert torch.equal(out_k, buf.k_cache.cpu()) and torch.equal(out_v, buf.v_cache.cpu())
    assert torch.equal(out_o, buf.origin.cpu())


def test_host_prefill_chained_calls(cuda):
    """HostPrefill.run(join=False) back to back on two Q/K/V sets: each host output set equals its device result."""
    sizes, n_q, n_kv, rho = [1024, 777, 1024, 1024], 28, 4, 0.5
    plan = qp.GroupPlan.from_sizes(sizes, rho)
    g = plan.to(cuda)
    hp = qp.HostPrefill(plan, n_q, n_kv, 128, rho, cuda, chunks=2)
    ins, outs, refs = [], [], []
    for s in (0, 10):
        q = synth_groups(sizes, n_q, 128, 3 + s, False, cuda)
        k = synth_groups(sizes, n_kv, 128, 1 + s, True, cuda)
        v = synth_groups(sizes, n_kv, 128, 2 + s, False, cuda)
        buf = qp.prefill_layer(q, k, v, g, n_q, n_kv, rho)
        refs.append((buf.k_cache.cpu(), buf.v_cache.cpu(), buf.origin.cpu()))
        ins.append(tuple(t.cpu().pin_memory() for t in (q, k, v)))
        ok = torch.empty(hp.k_cache.numel(), dtype=torch.bfloat16).pin_memory()
        outs.append((ok, torch.empty_like(ok).pin_memory(),
                     torch.empty(hp.origin.numel(), dtype=torch.int64).pin_memory()))
    torch.cuda.synchronize()
    for (hq, hk, hv), (ok, ov, oo) in zip(ins, outs):
        hp.run(hq, hk, hv, ok, ov, oo, join=False)
    hp.join()
    torch.cuda.synchronize()
    for (ok, ov, oo), (rk, rv, ro) in zip(outs, refs):
        assert torch.equal(ok, rk) and torch.equal(ov, rv) and torch.equal(oo, ro)


def test_project_qkv_one_sm_variant(cuda, tmp_path):
    """The 1-SM GEMM variant (QVK_PROJ_2SM=0) and the opt-in 256 x 512 pair-tile variant (QVK_PROJ_WIDE=1; knobs are
    read once per process: one subprocess each) agree with the default 2-SM kernel — the wide one bit for bit (same
    per-element accumulation order), the 1-SM one within the bf16 tolerance — and their fused key-norm equals
    qvk_score on their own K bit for bit."""
    import subprocess
    import sys
    code = r"""
import math, sys, torch
sys.path.insert(0, %r)
import paper_2505_16175_b200 as qp
dev = torch.device('cuda', 0)
sizes = [1000, 777]
plan = qp.GroupPlan.from_sizes(sizes, 0.5); g = plan.to(dev); T = sum(sizes)
x = qp.synth_bf16(5, 7, 0, 0, T, 1, 1024, False, dev).view(T, 1024)
w = (qp.synth_bf16(5, 8, 0, 0, 8 * 128, 1, 1024, False, dev).float() / 32).to(torch.bfloat16).view(-1, 1024)
q, k, v, sc = qp.project_qkv(x, w, 4, 2, 128, g, with_scores=True)
assert sc.cpu().numpy().tobytes() == qp.score(k, v, g, 2, 128, qp.Scorer.key_norm_small).cpu().numpy().tobytes()
torch.save({'q': q.cpu(), 'k': k.cpu(), 'v': v.cpu()}, %r)
"""
    outs = []
    for i, knobs in enumerate(({"QVK_PROJ_2SM": "0"}, {"QVK_PROJ_2SM": "1"}, {"QVK_PROJ_WIDE": "1"})):
        path = tmp_path / f"p{i}.pt"
        env = dict(__import__("os").environ, **knobs)
        r = subprocess.run([sys.executable, "-c", code % (str(GOLD.parent.parent), str(path))], env=env,
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(torch.load(path))
    for name in ("q", "k", "v"):
        check_tol(outs[0][name], outs[1][name], f"1-SM vs 2-SM {name}")
        assert torch.equal(outs[1][name], outs[2][name]), f"wide vs 2-SM {name}"


@pytest.mark.parametrize("scorer,per_head", [(qp.Scorer.snapkv, True), (qp.Scorer.value_norm, True),
                                             (qp.Scorer.key_norm_small, False)])
def test_prefill_layer_x_other_scorers(cuda, scorer, per_head):
    """qvk_prefill_layer_x without the fused key-norm (SnapKV, value-norm, per-token pruning) == projection followed
    by qvk_prefill_layer, bit for bit; ragged groups."""
    sizes, d_model, n_q, n_kv, d_h, rho = [1024, 700, 1024], 1024, 8, 2, 128, 0.25
    T = sum(sizes)
    plan = qp.GroupPlan.from_sizes(sizes, rho)
    g = plan.to(cuda)
    x, w = _proj_inputs(T, d_model, n_q, n_kv, d_h, cuda, seed=13)
    buf, _ = qp.prefill_layer_x(x, w, g, n_q, n_kv, d_h, rho, scorer, per_head)
    q, k, v = qp.project_qkv(x, w, n_q, n_kv, d_h)
    buf2 = qp.prefill_layer(q, k, v, g, n_q, n_kv, rho, scorer, per_head)
    torch.cuda.synchronize()
    assert torch.equal(buf.o, buf2.o)
    assert torch.equal(buf.k_cache, buf2.k_cache) and torch.equal(buf.v_cache, buf2.v_cache)
    assert torch.equal(buf.origin, buf2.origin)


def test_frame_prefill_ragged_last_group(cuda):
    """FramePrefill with a frame count that leaves a short last group (prefill.cpp:170-183) == device path."""
    F, fpg, tpf, H, W = 23, 4, 64, 64, 64
    n_q, n_kv, d_h, d_model, rho = 8, 2, 128, 512, 0.5
    plan = qp.GroupPlan.plan(F, fpg, tpf, rho, 1)
    assert int(plan.sizes[-1]) == 3 * tpf
    g = plan.to(cuda)
    fr = _frames(F, H, W, cuda, seed=9)
    embed = ((torch.rand(d_model, 3, generator=torch.Generator().manual_seed(5)) * 2 - 1) / 255).to(cuda)
    w = (torch.randn((n_q + 2 * n_kv) * d_h, d_model, generator=torch.Generator().manual_seed(6)) /
         math.sqrt(d_model)).to(torch.bfloat16).to(cuda)
    buf, _ = qp.prefill_layer_x(qp.tokenize(fr, tpf, embed, bf16=True), w, g, n_q, n_kv, d_h, rho)
    fp = qp.FramePrefill(plan, tpf, H, W, embed, w, n_q, n_kv, d_h, rho, cuda, chunks=4)
    hf = fr.cpu().pin_memory()
    out_k = torch.empty(fp.k_cache.numel(), dtype=torch.bfloat16).pin_memory()
    out_v = torch.empty_like(out_k).pin_memory()
    out_o = torch.empty(fp.origin.numel(), dtype=torch.int64).pin_memory()
    fp.run(hf, out_k, out_v, out_o)
    torch.cuda.synchronize()
    assert torch.equal(out_k, buf.k_cache.cpu()) and torch.equal(out_v, buf.v_cache.cpu())
    assert torch.equal(out_o, buf.origin.cpu())


def test_streaming_prefill_overlaps_a_slow_producer(cuda):
    """Overlap pipeline: groups submitted by a producer thread as they are 'decoded' (a fixed delay per group), in
    a shuffled order; the result equals the batch path, and the wall time stays close to the producer's time (the
    GPU work of group g hides under the decoding of group g + 1)."""
    import threading
    import time
    F, fpg, tpf, H, W = 32, 4, 64, 64, 64
    n_q, n_kv, d_h, d_model, rho = 8, 2, 128, 512, 0.5
    plan = qp.GroupPlan.plan(F, fpg, tpf, rho, 1)
    g = plan.to(cuda)
    fr = _frames(F, H, W, cuda, seed=21)
    embed = ((torch.rand(d_model, 3, generator=torch.Generator().manual_seed(8)) * 2 - 1) / 255).to(cuda)
    w = (torch.randn((n_q + 2 * n_kv) * d_h, d_model, generator=torch.Generator().manual_seed(9)) /
         math.sqrt(d_model)).to(torch.bfloat16).to(cuda)
    buf, _ = qp.prefill_layer_x(qp.tokenize(fr, tpf, embed, bf16=True), w, g, n_q, n_kv, d_h, rho)
    hf = fr.cpu().pin_memory()
    sp = qp.StreamingPrefill(plan, tpf, H, W, embed, w, n_q, n_kv, d_h, rho, cuda)
    order = [3, 0, 7, 1, 6, 2, 5, 4]
    delay = 0.02
    ready = []
    cv = threading.Condition()

    def producer():
        for gi in order:
            time.sleep(delay)  # "decode" the group's frames
            with cv:
                ready.append(gi)
                cv.notify()

    t = threading.Thread(target=producer)
    t0 = time.perf_counter()
    t.start()
    done = 0
    while done < len(order):
        with cv:
            while len(ready) <= done:
                cv.wait()
            gi = ready[done]
        sp.submit(gi, hf[gi * fpg:(gi + 1) * fpg])
        done += 1
    out_k = torch.empty(sp.k_cache.numel(), dtype=torch.bfloat16).pin_memory()
    out_v = torch.empty_like(out_k).pin_memory()
    out_o = torch.empty(sp.origin.numel(), dtype=torch.int64).pin_memory()
    sp.finish(out_k, out_v, out_o)
    wall = time.perf_counter() - t0
    t.join()
    assert torch.equal(out_k, buf.k_cache.cpu()) and torch.equal(out_v, buf.v_cache.cpu())
    assert torch.equal(out_o, buf.origin.cpu())
    assert wall < len(order) * delay + 0.5, wall  # prefill hidden under the producer (plus a first-launch margin)


def test_reserve_sms_leaves_results_unchanged(cuda):
    """qvk_reserve_sms shrinks the persistent grids (attention, projection) for work running beside them (the N > 1
    all-gather's NCCL CTAs); each work unit is computed the same way whatever CTA runs it, so outputs are
    bit-identical with and without a reservation."""
    sizes, n_q, n_kv, d = [1024, 700, 4096], 28, 4, 128
    plan = qp.GroupPlan.from_sizes(sizes, 0.5)
    g = plan.to(cuda)
    q = torch.cat([qp.synth_bf16(9, 3, 0, i, n, n_q, d, False, cuda) for i, n in enumerate(sizes)])
    k = torch.cat([qp.synth_bf16(9, 1, 0, i, n, n_kv, d, True, cuda) for i, n in enumerate(sizes)])
    v = torch.cat([qp.synth_bf16(9, 2, 0, i, n, n_kv, d, False, cuda) for i, n in enumerate(sizes)])
    x, w = _proj_inputs(sum(sizes), 1024, n_q, n_kv, d, cuda)
    outs = []
    for n in (0, 20, 0):
        qp.reserve_sms(n)
        try:
            o = qp.attention(q, k, v, g, n_q, n_kv, 1 / math.sqrt(d))
            pq, pk, pv = qp.project_qkv(x, w, n_q, n_kv, d)
            torch.cuda.synchronize()
        finally:
            qp.reserve_sms(0)
        outs.append((o, pq, pk, pv))
    for a, b in zip(outs[0], outs[1]):
        assert torch.equal(a, b)
    with pytest.raises(qp.QvError):
        qp.reserve_sms(-1)
    with pytest.raises(qp.QvError):
        qp.reserve_sms(100000)
