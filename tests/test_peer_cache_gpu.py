"""GPU: the cache all-gather fused into the compaction (distributed.PeerCache + qvk_prefill_layer_dests).

Two ranks share the one GPU of the test box (CUDA IPC maps each rank's cache into the other process exactly as it
maps a peer GPU's over NVLink); the handles are exchanged over gloo.  Every rank prefills its own block of groups and
its fused prune stores each retained row into BOTH ranks' caches; after the fence each rank must hold the complete
pruned cache, bit-identical to a single-rank prefill of all groups.
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q_out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2505_16175_b200 as qp
        from paper_2505_16175_b200.distributed import PeerCache

        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        frames, fpg, tpf, n_q, n_kv, d, rho = 40, 4, 128, 8, 2, 128, 0.5   # 10 groups of 512 tokens, ragged split
        plan = qp.GroupPlan.plan(frames, fpg, tpf, rho, world)
        shard = plan.shard(rank, world)
        a = int(plan.rank_begin[rank])
        sizes = [int(s) for s in shard.sizes]
        mk = lambda tag, h, hs: torch.cat([qp.synth_bf16(1, tag, 0, a + i, n, h, d, hs, dev)  # noqa: E731
                                           for i, n in enumerate(sizes)])
        q, k, v = mk(3, n_q, False), mk(1, n_kv, True), mk(2, n_kv, False)
        buf = qp.LayerBuffers.allocate(shard, n_q, n_kv, d, True, dev, cache_rows=plan.total_rows)
        buf.k_cache.zero_()
        buf.v_cache.zero_()
        buf.origin.zero_()
        peers = PeerCache([buf.k_cache, buf.v_cache, buf.origin])
        qp.prefill_layer_dests(q, k, v, shard.to(dev), n_q, n_kv, rho, peers, buf, cache_row_offset=shard.row_base)
        peers.fence(dev)
        # reference: one rank prefills every group
        full = qp.GroupPlan.plan(frames, fpg, tpf, rho, 1)
        fs = [int(s) for s in full.sizes]
        rq = torch.cat([qp.synth_bf16(1, 3, 0, i, n, n_q, d, False, dev) for i, n in enumerate(fs)])
        rk = torch.cat([qp.synth_bf16(1, 1, 0, i, n, n_kv, d, True, dev) for i, n in enumerate(fs)])
        rv = torch.cat([qp.synth_bf16(1, 2, 0, i, n, n_kv, d, False, dev) for i, n in enumerate(fs)])
        ref = qp.prefill_layer(rq, rk, rv, full.to(dev), n_q, n_kv, rho)
        torch.cuda.synchronize()
        ok = (torch.equal(buf.k_cache, ref.k_cache) and torch.equal(buf.v_cache, ref.v_cache)
              and torch.equal(buf.origin, ref.origin))
        dist.barrier()
        peers.close()
        q_out.put((rank, ok, None))
    except Exception as e:  # noqa: BLE001
        q_out.put((rank, False, repr(e)))
    finally:
        dist.destroy_process_group()


def test_fused_allgather_two_ranks_one_gpu():
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
