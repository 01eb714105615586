"""GPU parity of the GQA attention_score scorer (include/qvk.h qvk_score_text).

The reference scores a token by the mean raw dot product of its key with every text-token query over every head
(prefill.cpp:213-230, MHA only).  Under GQA the device path pre-sums the text queries over the text tokens and the
query heads of each KV head (qbar, one fp32 row per KV head) and then runs the reference's OWN sequential double dot
product on that single row — so the scores are compared, bit for bit, against the unmodified reference
(qvref::score_tokens, n_h = 1, on the pre-summed row) divided by T * n_q/n_kv (per head) or T * n_q (per token);
retained index sets, cache rows and origins are then bit-exact against the oracle's top-k on those scores.
"""
import numpy as np
import pytest
import torch

import paper_2505_16175_b200 as qp
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _inputs(sizes, n_q, n_kv, d, T, device, seed=5):
    k = torch.cat([qp.synth_bf16(seed, 1, 0, g, n, n_kv, d, True, device) for g, n in enumerate(sizes)])
    gen = torch.Generator().manual_seed(seed)
    tq = (torch.randn(T, n_q, d, generator=gen) * 0.5).to(device)
    return k, tq


def test_text_query_sum_bitexact(cuda):
    for n_q, n_kv, d, T in ((28, 4, 128, 7), (4, 2, 64, 1), (8, 8, 128, 3)):
        _, tq = _inputs([1], n_q, n_kv, d, T, cuda)
        got = qp.text_query_sum(tq, n_q, n_kv).cpu().numpy()
        want = O.text_query_sum(tq.cpu().numpy(), n_q, n_kv, d)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (n_q, n_kv, d, T)


@pytest.mark.parametrize("sizes,n_q,n_kv,d,T", [([300, 1000, 77], 28, 4, 128, 7), ([256, 256], 4, 2, 64, 16),
                                                ([4096], 28, 4, 128, 64), ([1, 5], 8, 2, 128, 2)])
@pytest.mark.parametrize("per_head", [True, False])
def test_score_text_matches_reference(cuda, sizes, n_q, n_kv, d, T, per_head):
    k, tq = _inputs(sizes, n_q, n_kv, d, T, cuda)
    plan = qp.GroupPlan.from_sizes(sizes, 0.5)
    got = qp.score_text(k, plan.to(cuda), tq, n_q, n_kv, per_head).cpu().numpy()
    qbar = O.text_query_sum(tq.cpu().numpy(), n_q, n_kv, d)
    kf = k.float().cpu().numpy()
    heads = n_kv if per_head else 1
    t0 = 0
    for n in sizes:
        want = O.score_text_ref(kf[t0:t0 + n], n, n_q, n_kv, d, per_head, qbar, T)
        seg = got[heads * t0: heads * (t0 + n)].reshape(heads, n)
        assert np.array_equal(seg.view(np.uint64), want.view(np.uint64)), "scores differ from the reference"
        t0 += n


@pytest.mark.parametrize("per_head", [True, False])
def test_prefill_layer_attention_score(cuda, per_head):
    """qvk_prefill_layer with the text query in qvk_layer_params: attention, scores, top-k, cache — bit-exact against
    the reference's scores and the oracle's top-k / gather."""
    sizes, n_q, n_kv, d, T, rho = [1024, 700, 4096], 28, 4, 128, 16, 0.25
    k, tq = _inputs(sizes, n_q, n_kv, d, T, cuda)
    q = torch.cat([qp.synth_bf16(5, 3, 0, g, n, n_q, d, False, cuda) for g, n in enumerate(sizes)])
    v = torch.cat([qp.synth_bf16(5, 2, 0, g, n, n_kv, d, False, cuda) for g, n in enumerate(sizes)])
    plan = qp.GroupPlan.from_sizes(sizes, rho)
    buf = qp.prefill_layer(q, k, v, plan.to(cuda), n_q, n_kv, rho, qp.Scorer.attention_score, per_head,
                           text_query=tq)
    torch.cuda.synchronize()
    assert qp.last_prune_route() in (1, 3)
    heads, width = (n_kv, d) if per_head else (1, n_kv * d)
    qbar = O.text_query_sum(tq.cpu().numpy(), n_q, n_kv, d)
    kf, vf = k.float().cpu().numpy(), v.float().cpu().numpy()
    idx = buf.idx[: plan.total_rows * heads].view(-1, heads).cpu().numpy()
    kc = buf.k_cache.view(-1, heads, width).float().cpu().numpy()
    vc = buf.v_cache.view(-1, heads, width).float().cpu().numpy()
    org = buf.origin.view(-1, heads).cpu().numpy()
    t0 = 0
    for gi, n in enumerate(sizes):
        r0, kk = plan.row_off[gi], plan.keep[gi]
        sc = O.score_text_ref(kf[t0:t0 + n], n, n_q, n_kv, d, per_head, qbar, T)
        want = O.select_heads(sc, n, heads, kk)
        assert np.array_equal(idx[r0:r0 + kk], want), f"group {gi}: retained index sets differ"
        kh = kf[t0:t0 + n].reshape(n, heads, width)
        vh = vf[t0:t0 + n].reshape(n, heads, width)
        assert np.array_equal(kc[r0:r0 + kk], O.gather_heads(kh, heads, width, want))
        assert np.array_equal(vc[r0:r0 + kk], O.gather_heads(vh, heads, width, want))
        assert np.array_equal(org[r0:r0 + kk], want.astype(np.int64) + t0)
        t0 += n


def test_attention_score_requires_text_query(cuda):
    sizes, n_q, n_kv, d = [256], 4, 2, 64
    k, _ = _inputs(sizes, n_q, n_kv, d, 1, cuda)
    q = torch.cat([qp.synth_bf16(5, 3, 0, 0, 256, n_q, d, False, cuda)])
    plan = qp.GroupPlan.from_sizes(sizes, 0.5)
    with pytest.raises(qp.QvError, match="attention_score scorer requires a text query"):
        qp.prefill_layer(q, k, k, plan.to(cuda), n_q, n_kv, 0.5, qp.Scorer.attention_score, True)
    with pytest.raises(qp.QvError, match="attention_score scorer requires a text query"):
        qp.score_text(k, plan.to(cuda), None, n_q, n_kv, True)
