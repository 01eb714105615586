"""Multi-rank group sharding on CPU: world size 2 over gloo.

Each rank takes its contiguous block of groups from GroupPlan.plan(..., world).shard(rank), prunes them (here with
the oracle, since this container has no GPU — the device path is covered by tests/test_kernels_gpu.py), writes the
pruned rows at their GLOBAL cache offsets, and allgather_cache replicates the cache.  The replicated cache must be
bit-identical to the single-rank (P = 1) result, including ragged last groups and uneven rank splits.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2505_16175_b200 as qp
from oracle import oracle as O
from paper_2505_16175_b200.distributed import allgather_cache, segment_bounds

N_KV, D = 2, 16


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _pruned_cache(plan, groups, k, v, rho):
    """Oracle prune of `groups` (global indices) into full-size cache buffers at the global offsets."""
    R = plan.total_rows
    kc = np.zeros((R, N_KV, D), np.float32)
    vc = np.zeros((R, N_KV, D), np.float32)
    org = np.zeros((R, N_KV), np.int64)
    for gi in groups:
        t0, t1 = plan.tok_off[gi], plan.tok_off[gi + 1]
        n, keep, r0 = t1 - t0, plan.keep[gi], plan.row_off[gi]
        idx = O.select_heads(O.score_norm(k[t0:t1], N_KV, D, True), n, N_KV, keep)  # (keep, heads)
        kc[r0:r0 + keep] = O.gather_heads(k[t0:t1], N_KV, D, idx)
        vc[r0:r0 + keep] = O.gather_heads(v[t0:t1], N_KV, D, idx)
        org[r0:r0 + keep] = plan.first_token[gi].astype(np.int64) + idx
    return kc, vc, org


def _inputs(plan):
    T = plan.total_tokens
    k = O.bf16_to_f32(O.synth_bf16(1, 1, 0, 0, T, N_KV, D, True)).reshape(T, N_KV, D)
    v = O.bf16_to_f32(O.synth_bf16(1, 2, 0, 0, T, N_KV, D, False)).reshape(T, N_KV, D)
    return k, v


def _worker(rank, world, port, frames, fpg, tpf, rho, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = qp.GroupPlan.plan(frames, fpg, tpf, rho, world)
        shard = plan.shard(rank, world)
        a, b = int(plan.rank_begin[rank]), int(plan.rank_begin[rank + 1])
        assert shard.n_groups == b - a and shard.row_base == int(plan.row_off[a])
        k, v = _inputs(plan)
        kc, vc, org = _pruned_cache(plan, range(a, b), k, v, rho)
        tensors = [torch.from_numpy(kc.reshape(-1)), torch.from_numpy(vc.reshape(-1)),
                   torch.from_numpy(org.reshape(-1))]
        allgather_cache(tensors, segment_bounds(plan, world), [N_KV * D, N_KV * D, N_KV])
        if rank == 0:
            np.savez(out_path, k=tensors[0].numpy(), v=tensors[1].numpy(), o=tensors[2].numpy())
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("frames,fpg,tpf,rho", [(37, 4, 16, 0.5), (64, 16, 8, 0.25), (9, 1, 33, 0.125)])
def test_two_rank_cache_equals_single_rank(tmp_path, frames, fpg, tpf, rho):
    world = 2
    out = tmp_path / "cache.npz"
    mp.start_processes(_worker, args=(world, _free_port(), frames, fpg, tpf, rho, str(out)), nprocs=world,
                       join=True, start_method="spawn")
    plan = qp.GroupPlan.plan(frames, fpg, tpf, rho, 1)
    k, v = _inputs(plan)
    kc, vc, org = _pruned_cache(plan, range(plan.n_groups), k, v, rho)
    got = np.load(out)
    assert got["k"].tobytes() == kc.reshape(-1).tobytes()
    assert got["v"].tobytes() == vc.reshape(-1).tobytes()
    assert got["o"].tobytes() == org.reshape(-1).tobytes()


def test_partition_is_balanced_and_contiguous():
    plan = qp.GroupPlan.plan(3600, 16, 256, 0.5, 8)  # C4: 225 groups over 8 ranks
    rb = plan.rank_begin
    assert rb[0] == 0 and rb[-1] == plan.n_groups and np.all(np.diff(rb) >= 0)
    counts = np.diff(rb)
    assert counts.max() - counts.min() <= 1
    bounds = segment_bounds(plan, 8)
    assert bounds[0][0] == 0 and bounds[-1][1] == plan.total_rows
    assert all(bounds[i][1] == bounds[i + 1][0] for i in range(7))
