"""GPU: the multi-GPU cache assembly.

* qvk_allgather_layer through the C ABI's NCCL communicator (qvk_comm_*): a world-size-1 communicator on the test
  box's one GPU runs the real grouped ncclBroadcast launch (NCCL refuses two ranks on one device, so larger worlds
  need the 8-GPU box: bench.py --gpus N);
* two ranks sharing the GPU run the PRODUCT kernels (qvk_prefill_layer) on their own block of groups, write the
  pruned rows at their global cache offsets and replicate the cache (torch.distributed broadcasts over gloo): the
  replicated cache must be bit-identical to a single-rank prefill of every group.
"""
import ctypes as C
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2505_16175_b200 as qp
from paper_2505_16175_b200._lib import check, lib

pytestmark = pytest.mark.gpu


def test_nccl_world_one_allgather(cuda):
    uid = (C.c_char * 128)()
    check(lib.qvk_comm_unique_id(uid))
    comm = C.c_void_p(0)
    check(lib.qvk_comm_init(C.byref(comm), 1, 0, uid))
    r, w = C.c_int32(-1), C.c_int32(-1)
    check(lib.qvk_comm_rank(comm, C.byref(r), C.byref(w)))
    assert (r.value, w.value) == (0, 1)
    rows, heads, width = 1000, 4, 128
    kc = torch.randn(rows * heads * width, device=cuda).to(torch.bfloat16)
    vc = torch.randn(rows * heads * width, device=cuda).to(torch.bfloat16)
    og = torch.arange(rows * heads, device=cuda, dtype=torch.int64)
    before = (kc.clone(), vc.clone(), og.clone())
    seg = (C.c_int64 * 2)(0, rows)
    check(lib.qvk_allgather_layer(torch.cuda.current_stream().cuda_stream, comm, seg, heads, width, kc.data_ptr(),
                                  vc.data_ptr(), og.data_ptr()))
    torch.cuda.synchronize()
    check(lib.qvk_comm_check(comm))
    assert torch.equal(kc, before[0]) and torch.equal(vc, before[1]) and torch.equal(og, before[2])
    bad = (C.c_int64 * 2)(5, 2)
    assert lib.qvk_allgather_layer(None, comm, bad, heads, width, kc.data_ptr(), vc.data_ptr(), None) == -1
    check(lib.qvk_comm_destroy(comm))


def test_nccl_cta_cap_reserves_sms(cuda):
    """QVK_COMM_CTAS: qvk_comm_init caps NCCL's CTAs (ncclConfig_t.maxCTAs) and reserves as many SMs from the
    persistent kernels' grids until qvk_comm_destroy (a world-1 communicator with the cap set explicitly — at
    world > 1 it is on by default)."""
    import subprocess
    import sys
    code = r"""
import ctypes as C, sys, torch
sys.path.insert(0, %r)
import paper_2505_16175_b200 as qp
from paper_2505_16175_b200._lib import check, lib
torch.zeros(1, device='cuda')
uid = (C.c_char * 128)(); check(lib.qvk_comm_unique_id(uid))
comm = C.c_void_p(0); check(lib.qvk_comm_init(C.byref(comm), 1, 0, uid))
assert qp.reserve_sms(6) == 6            # the communicator's reservation was active
qp.reserve_sms(6)
rows, heads, width = 512, 2, 128
kc = torch.randn(rows * heads * width, device='cuda').to(torch.bfloat16); ref = kc.clone()
seg = (C.c_int64 * 2)(0, rows)
check(lib.qvk_allgather_layer(torch.cuda.current_stream().cuda_stream, comm, seg, heads, width, kc.data_ptr(),
                              kc.data_ptr(), None))
torch.cuda.synchronize(); check(lib.qvk_comm_check(comm))
assert torch.equal(kc, ref)
check(lib.qvk_comm_destroy(comm))
assert qp.reserve_sms(0) == 0            # released by qvk_comm_destroy
print("ok")
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, QVK_COMM_CTAS="6")
    r = subprocess.run([sys.executable, "-c", code % root], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q_out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2505_16175_b200.distributed import allgather_cache, segment_bounds

        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        frames, fpg, tpf, n_q, n_kv, d, rho = 44, 4, 128, 8, 2, 128, 0.5   # 11 groups of 512 tokens, ragged split
        plan = qp.GroupPlan.plan(frames, fpg, tpf, rho, world)
        shard = plan.shard(rank, world)
        a = int(plan.rank_begin[rank])
        sizes = [int(s) for s in shard.sizes]
        mk = lambda tag, h, hs: torch.cat([qp.synth_bf16(1, tag, 0, a + i, n, h, d, hs, dev)  # noqa: E731
                                           for i, n in enumerate(sizes)])
        q, k, v = mk(3, n_q, False), mk(1, n_kv, True), mk(2, n_kv, False)
        buf = qp.LayerBuffers.allocate(shard, n_q, n_kv, d, True, dev, cache_rows=plan.total_rows)
        for t in (buf.k_cache, buf.v_cache, buf.origin):
            t.zero_()
        qp.prefill_layer(q, k, v, shard.to(dev), n_q, n_kv, rho, buffers=buf, cache_row_offset=shard.row_base)
        torch.cuda.synchronize()
        allgather_cache([buf.k_cache, buf.v_cache, buf.origin], segment_bounds(plan, world),
                        [n_kv * d, n_kv * d, n_kv])
        torch.cuda.synchronize()
        full = qp.GroupPlan.plan(frames, fpg, tpf, rho, 1)
        fs = [int(s) for s in full.sizes]
        rq = torch.cat([qp.synth_bf16(1, 3, 0, i, n, n_q, d, False, dev) for i, n in enumerate(fs)])
        rk = torch.cat([qp.synth_bf16(1, 1, 0, i, n, n_kv, d, True, dev) for i, n in enumerate(fs)])
        rv = torch.cat([qp.synth_bf16(1, 2, 0, i, n, n_kv, d, False, dev) for i, n in enumerate(fs)])
        ref = qp.prefill_layer(rq, rk, rv, full.to(dev), n_q, n_kv, rho)
        torch.cuda.synchronize()
        ok = (torch.equal(buf.k_cache, ref.k_cache) and torch.equal(buf.v_cache, ref.v_cache)
              and torch.equal(buf.origin, ref.origin))
        q_out.put((rank, ok, None))
    except Exception as e:  # noqa: BLE001
        q_out.put((rank, False, repr(e)))
    finally:
        dist.destroy_process_group()


def test_two_ranks_product_kernels_allgather():
    ctx = mp.get_context("spawn")
    q_out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q_out)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q_out.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, err in sorted(res):
        assert err is None, f"rank {rank}: {err}"
        assert ok, f"rank {rank}: replicated cache differs from the single-rank prefill"
