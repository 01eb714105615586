"""Multi-GPU group sharding (north star: "groups shard naturally across the 8 GPUs ... a single NCCL all-gather over
NVLink assembles the pruned cache").

Every rank prefills and prunes the contiguous block of groups GroupPlan.plan(..., world).shard(rank) gives it and
writes the pruned rows at their GLOBAL cache offsets (cache row offsets are a pure function of (rho, N_g),
prefill.cpp:235-238, so no exchange is needed before the collective).  The one data-path collective is the
all-gather of the pruned K/V/origin segments; NCCL's all-gather needs equal counts, the per-rank segments are ragged
(225 groups over 8 ranks), so it is issued as one broadcast per source rank directly into that rank's slice of the
replicated cache (no padding, no compaction copy), grouped so NCCL overlaps them.
Works on any torch.distributed backend (gloo for the CPU tests, nccl on the GPU box).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .prefill import GroupPlan


def segment_bounds(plan: GroupPlan, world: int) -> list[tuple[int, int]]:
    """Global cache rows [begin, end) owned by each rank."""
    rb = plan.rank_begin
    if len(rb) != world + 1:
        raise ValueError("plan was built for a different world size")
    return [(int(plan.row_off[rb[r]]), int(plan.row_off[rb[r + 1]])) for r in range(world)]


def allgather_cache(tensors: list[torch.Tensor], bounds: list[tuple[int, int]], unit: list[int], group=None,
                    async_op: bool = False):
    """Replicate each rank's pruned segment into every rank's full cache.

    tensors[i] is a flat cache buffer whose row r occupies [r*unit[i], (r+1)*unit[i]); on entry each rank has filled
    its own rows bounds[rank]; on return (or after the returned work handles complete) every rank holds all rows.
    """
    world = len(bounds)
    if world == 1:
        return []
    works = []
    for t, u in zip(tensors, unit):
        for src, (b, e) in enumerate(bounds):
            if e > b:
                works.append(dist.broadcast(t[b * u:e * u], src=src, group=group, async_op=True))
    if async_op:
        return works
    for w in works:
        w.wait()
    return []


class NcclComm:
    """The C ABI's NCCL communicator (qvk_comm_*, include/qvk.h) bootstrapped over torch.distributed: rank 0 creates
    the ncclUniqueId, the process group ships it, every rank joins on its current device.  `allgather` replicates a
    layer's pruned cache with ONE grouped NCCL call (qvk_allgather_layer: an in-place broadcast per source rank and
    buffer inside one ncclGroupStart/End) on the given stream."""

    def __init__(self, group=None):
        import ctypes as C

        from ._lib import check, lib

        self._C, self._lib, self._check = C, lib, check
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        uid = (C.c_char * 128)()
        if self.rank == 0:
            check(lib.qvk_comm_unique_id(uid))
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=0, group=group)
        self.comm = C.c_void_p(0)
        check(lib.qvk_comm_init(C.byref(self.comm), self.world, self.rank, C.create_string_buffer(box[0], 128)))

    def allgather(self, k_cache: torch.Tensor, v_cache: torch.Tensor, origin: torch.Tensor | None,
                  bounds: list[tuple[int, int]], heads: int, width: int, stream=None) -> None:
        C = self._C
        rb = (C.c_int64 * (self.world + 1))(*([b for b, _ in bounds] + [bounds[-1][1]]))
        s = (stream or torch.cuda.current_stream()).cuda_stream
        self._check(self._lib.qvk_allgather_layer(s, self.comm, rb, heads, width, k_cache.data_ptr(),
                                                  v_cache.data_ptr(), None if origin is None else origin.data_ptr()))

    def check(self) -> None:
        self._check(self._lib.qvk_comm_check(self.comm))

    def close(self) -> None:
        if self.comm:
            self._check(self._lib.qvk_comm_destroy(self.comm))
            self.comm = self._C.c_void_p(0)


class PeerCache:
    """The cache all-gather fused into the compaction: every rank maps the other ranks' cache buffers into its address
    space (CUDA IPC over NVLink; qvk_ipc_*) and the fused prune kernel stores each retained row into ALL ranks' caches
    (qvk_prefill_layer_dests / qvk_prune_dests), so the pruned cache is replicated as a side effect of the compaction —
    no separate collective, the NVLink transfers overlap the kernel's own HBM traffic row by row.  After every rank's
    kernel, one cross-rank barrier (`fence`) makes the replicated cache safe to read.

    tensors: this rank's cache buffers (k_cache, v_cache, origin); the same-shaped buffers of every rank are mapped.
    """

    def __init__(self, tensors: list[torch.Tensor], group=None):
        import ctypes as C

        from ._lib import check, lib

        self._lib, self._check = lib, check
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if self.world > 8:
            raise ValueError("PeerCache: at most 8 ranks (destinations per row)")
        self.group = group
        handles = []
        for t in tensors:
            h = (C.c_char * 64)()
            off = C.c_uint64(0)
            check(lib.qvk_ipc_get_handle(t.data_ptr(), h, C.byref(off)))
            handles.append((bytes(h), off.value))
        gathered = [None] * self.world
        dist.all_gather_object(gathered, handles, group=group)
        self._bases = []
        self.ptrs = []  # per tensor: [own, then the other ranks in rank order]
        for i, t in enumerate(tensors):
            row = [t.data_ptr()]
            for r in range(self.world):
                if r == self.rank:
                    continue
                base = C.c_void_p(0)
                hb, off = gathered[r][i]
                check(lib.qvk_ipc_open(C.create_string_buffer(hb, 64), C.byref(base)))
                self._bases.append(base.value)
                row.append(base.value + off)
            self.ptrs.append(row)
        self.arrays = [(C.c_void_p * len(row))(*row) for row in self.ptrs]
        # device-side barrier state: one 32-bit counter per rank (IPC-mapped by the others) and an error word
        dev = tensors[0].device
        self.flag = torch.zeros(64, dtype=torch.int32, device=dev)  # own 256-byte slot, counter at [0]
        self.err = torch.zeros(1, dtype=torch.int32, device=dev)
        h = (C.c_char * 64)()
        off = C.c_uint64(0)
        torch.cuda.synchronize(dev)
        check(lib.qvk_ipc_get_handle(self.flag.data_ptr(), h, C.byref(off)))
        fl = [None] * self.world
        dist.all_gather_object(fl, (bytes(h), off.value), group=group)
        flags = []
        for r in range(self.world):
            if r == self.rank:
                flags.append(self.flag.data_ptr())
                continue
            base = C.c_void_p(0)
            check(lib.qvk_ipc_open(C.create_string_buffer(fl[r][0], 64), C.byref(base)))
            self._bases.append(base.value)
            flags.append(base.value + fl[r][1])
        self._flags = (C.c_void_p * self.world)(*flags)
        self.epoch = 0
        dist.barrier(group=group)  # every rank mapped every counter before the first fence

    def fence(self, device=None):
        """Cross-rank barrier after this step's kernels, ON THE DEVICE (qvk_peer_barrier): stream-ordered after the
        prune, so later work on the stream sees every peer's stores into our cache; no host synchronisation."""
        self.epoch += 1
        s = torch.cuda.current_stream(device).cuda_stream
        self._check(self._lib.qvk_peer_barrier(s, self.world, self._flags, self.rank, self.epoch,
                                               self.err.data_ptr()))

    def check(self) -> None:
        """Raise if a device barrier timed out (a peer never arrived)."""
        if int(self.err.item()):
            raise RuntimeError("PeerCache: a peer did not reach the device barrier (timeout)")

    def close(self):
        torch.cuda.synchronize()
        dist.barrier(group=self.group)  # no peer still stores into our buffers when they are unmapped
        for b in self._bases:
            self._check(self._lib.qvk_ipc_close(b))
        self._bases = []
