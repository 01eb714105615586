"""The C ABI from plain C (examples/c_abi_prune.c: include/qvk.h only, gcc -std=c99): it compiles and links against
libqvk.so without CUDA headers (CPU), and on the GPU its prune of a small video equals the Python path's bit for bit."""
import os
import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest
import torch

import paper_2505_16175_b200 as qp

ROOT = Path(__file__).resolve().parent.parent
LIB = ROOT / "paper_2505_16175_b200" / "lib"


def _compile(tmp_path):
    if shutil.which("gcc") is None or not (LIB / "libqvk.so").exists():
        pytest.skip("gcc or libqvk.so missing")
    exe = tmp_path / "c_abi_prune"
    subprocess.run(["gcc", "-std=c99", "-O2", "-Wall", "-Werror", f"-I{ROOT / 'include'}",
                    str(ROOT / "examples" / "c_abi_prune.c"), f"-L{LIB}", "-lqvk", f"-Wl,-rpath,{LIB}", "-o",
                    str(exe)], check=True, capture_output=True, text=True)
    return exe


def test_c_example_compiles_and_links_without_cuda_headers(tmp_path):
    _compile(tmp_path)


def _lcg_bf16(n):
    """The example's inputs: one 64-bit LCG, alternating K / V draws, uniform [-1, 1) -> fp32 -> bf16 (RNE)."""
    s = 0x9e3779b97f4a7c15
    a, c, m = 6364136223846793005, 1442695040888963407, (1 << 64) - 1
    draws = np.empty(2 * n, dtype=np.float64)
    for i in range(2 * n):
        s = (s * a + c) & m
        draws[i] = (s >> 11) / 9007199254740992.0 * 2.0 - 1.0
    u = draws.astype(np.float32).view(np.uint32).astype(np.uint64)
    b = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    return b[0::2], b[1::2]


@pytest.mark.gpu
def test_c_example_matches_python_path(tmp_path):
    exe = _compile(tmp_path)
    out = tmp_path / "out.bin"
    r = subprocess.run([str(exe), str(out)], capture_output=True, text=True, env=dict(os.environ))
    assert r.returncode == 0, r.stderr
    frames, fpg, tpf, heads, width, rho = 16, 4, 64, 2, 128, 0.5
    plan = qp.GroupPlan.plan(frames, fpg, tpf, rho, 1)
    T, R = plan.total_tokens, plan.total_rows
    kb, vb = _lcg_bf16(T * heads * width)
    dev = torch.device("cuda", 0)
    k = torch.from_numpy(kb.view(np.int16)).view(torch.bfloat16).view(T, heads, width).to(dev)
    v = torch.from_numpy(vb.view(np.int16)).view(torch.bfloat16).view(T, heads, width).to(dev)
    kc, vc, origin, idx = qp.prune(k, v, plan.to(dev), heads, width, qp.Scorer.key_norm_small, rho)
    raw = out.read_bytes()
    c_idx = np.frombuffer(raw[:R * heads * 4], dtype=np.uint32)
    c_kc = np.frombuffer(raw[R * heads * 4:], dtype=np.uint16)
    assert np.array_equal(c_idx, idx[:R * heads].cpu().numpy().astype(np.uint32))
    assert np.array_equal(c_kc, kc.view(torch.int16).cpu().numpy().view(np.uint16))


@pytest.mark.gpu
@pytest.mark.parametrize("nbytes", [1, 4 << 20, (4 << 20) + 1, (32 << 20) + 12345, (100 << 20) + 7])
def test_pageable_staged_copies(cuda, nbytes):
    """qvk_memcpy_{h2d,d2h}_pageable: pageable host buffers through the pinned double-buffered staging, every chunk
    boundary case (direct small copy, exact chunk multiples, ragged tails), bit-exact round trip."""
    import numpy as np
    import torch

    import paper_2505_16175_b200 as qp
    from paper_2505_16175_b200._lib import check

    src = np.random.default_rng(nbytes % 1000).integers(0, 256, nbytes, dtype=np.uint8)
    dev = torch.empty(nbytes, dtype=torch.uint8, device=cuda)
    check(qp.lib.qvk_memcpy_h2d_pageable(dev.data_ptr(), src.ctypes.data, nbytes, None))
    assert np.array_equal(dev.cpu().numpy(), src)
    out = np.zeros(nbytes, np.uint8)
    check(qp.lib.qvk_memcpy_d2h_pageable(out.ctypes.data, dev.data_ptr(), nbytes, None))
    assert np.array_equal(out, src)


@pytest.mark.gpu
def test_context_api_matches_prefill_layer(cuda):
    """qvk_ctx_create / qvk_ctx_prefill_layer(_x): the plan and workspaces allocated once from HOST offsets give the
    same attention output and pruned cache as qvk_prefill_layer with caller-provided descriptors, layer after layer."""
    import ctypes as C

    import numpy as np
    import torch

    import paper_2505_16175_b200 as qp
    from paper_2505_16175_b200 import _lib as L
    from paper_2505_16175_b200._lib import check

    sizes, n_q, n_kv, d, rho = [1024, 300, 2048], 28, 4, 128, 0.25
    plan = qp.GroupPlan.from_sizes(sizes, rho, first_tokens=[5, 2000, 9000])
    prm = L.QvkLayerParams(n_q, n_kv, d, int(qp.Scorer.key_norm_small), 1, rho, 1.0 / d ** 0.5, 32, 1, None, 0)
    ctx = C.c_void_p(0)
    tok = np.ascontiguousarray(plan.tok_off, np.int64)
    ft = np.ascontiguousarray(plan.first_token, np.uint64)
    check(qp.lib.qvk_ctx_create(C.byref(ctx), C.byref(prm), len(sizes), tok.ctypes.data, ft.ctypes.data))
    try:
        desc = L.QvkGroups()
        check(qp.lib.qvk_ctx_groups(ctx, C.byref(desc)))
        assert (desc.n_groups, desc.total_tokens, desc.total_rows) == (3, plan.total_tokens, plan.total_rows)
        s = torch.cuda.current_stream().cuda_stream
        for layer in range(2):
            q = torch.cat([qp.synth_bf16(1, 3, layer, i, n, n_q, d, False, cuda) for i, n in enumerate(sizes)])
            k = torch.cat([qp.synth_bf16(1, 1, layer, i, n, n_kv, d, True, cuda) for i, n in enumerate(sizes)])
            v = torch.cat([qp.synth_bf16(1, 2, layer, i, n, n_kv, d, False, cuda) for i, n in enumerate(sizes)])
            ref = qp.prefill_layer(q, k, v, plan.to(cuda), n_q, n_kv, rho)
            o = torch.empty_like(q)
            kc, vc = torch.empty_like(ref.k_cache), torch.empty_like(ref.v_cache)
            og = torch.empty_like(ref.origin)
            check(qp.lib.qvk_ctx_prefill_layer(ctx, s, q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),
                                               kc.data_ptr(), vc.data_ptr(), og.data_ptr()))
            torch.cuda.synchronize()
            assert torch.equal(o, ref.o) and torch.equal(kc, ref.k_cache) and torch.equal(vc, ref.v_cache)
            assert torch.equal(og, ref.origin)
        # from hidden states
        d_model = n_q * d
        x = torch.cat([qp.synth_bf16(1, 7, 0, i, n, 1, d_model, False, cuda) for i, n in enumerate(sizes)]).view(-1, d_model)
        w = (qp.synth_bf16(1, 8, 0, 0, (n_q + 2 * n_kv) * d, 1, d_model, False, cuda).float() / d_model ** 0.5
             ).to(torch.bfloat16).view(-1, d_model)
        ref, _ = qp.prefill_layer_x(x, w, plan.to(cuda), n_q, n_kv, d, rho)
        T = plan.total_tokens
        qw, kw, vw = (torch.empty(T, h, d, dtype=torch.bfloat16, device=cuda) for h in (n_q, n_kv, n_kv))
        o = torch.empty(T, n_q, d, dtype=torch.bfloat16, device=cuda)
        kc, vc, og = torch.empty_like(ref.k_cache), torch.empty_like(ref.v_cache), torch.empty_like(ref.origin)
        check(qp.lib.qvk_ctx_prefill_layer_x(ctx, s, x.data_ptr(), d_model, w.data_ptr(), qw.data_ptr(), kw.data_ptr(),
                                             vw.data_ptr(), o.data_ptr(), kc.data_ptr(), vc.data_ptr(), og.data_ptr()))
        torch.cuda.synchronize()
        assert torch.equal(o, ref.o) and torch.equal(kc, ref.k_cache) and torch.equal(og, ref.origin)
    finally:
        check(qp.lib.qvk_ctx_destroy(ctx))
