// Multi-GPU cache assembly through NCCL: groups are independent and every cache
// offset is static, so each rank writes its own groups' pruned rows at their global offsets and ONE grouped NCCL
// call replicates the layer's cache on every GPU for the decode step.  NCCL has no all-gather-v: the ragged rank
// segments are moved by one in-place ncclBroadcast per (source rank, buffer) inside a single
// ncclGroupStart/ncclGroupEnd, which NCCL fuses into one launch over NVLink / NVSwitch.  Built against the NCCL that
// torch bundles (nvidia/nccl, 2.28) so a torch process loads one NCCL runtime.
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"

struct qvk_comm_st {
    ncclComm_t comm = nullptr;
    bool owned = true;
    int rank = 0, world = 1;
    int reserved = 0;  // SMs this communicator reserved (qvk_reserve_sms), released by qvk_comm_destroy
};

namespace qvk {
namespace {

int nccl_fail(ncclResult_t r, const char* what) {
    std::string msg = std::string("NCCL error in ") + what + ": " + ncclGetErrorString(r);
    const char* last = ncclGetLastError(nullptr);
    if (last && *last) msg += std::string(" (") + last + ")";
    set_error(msg);
    return r == ncclInvalidArgument || r == ncclInvalidUsage ? QVK_E_INVALID : QVK_E_CUDA;
}

#define QVK_NCCL(expr)                                            \
    do {                                                          \
        const ncclResult_t _r = (expr);                           \
        if (_r != ncclSuccess) return nccl_fail(_r, #expr);       \
    } while (0)

int fill_rank(qvk_comm_st* c) {
    QVK_NCCL(ncclCommUserRank(c->comm, &c->rank));
    QVK_NCCL(ncclCommCount(c->comm, &c->world));
    return QVK_OK;
}

}  // namespace
}  // namespace qvk

namespace qvk {
namespace {

// Device-side cross-rank barrier over peer memory (replaces a host stream synchronise + torch barrier after the
// fused prune's peer stores): every rank adds 1 to every rank's counter (system-scope atomics over NVLink, after a
// system fence that publishes this rank's earlier stores — stream order puts the prune before this kernel), then
// spins until its own counter reaches epoch * n.  A rank that never arrives trips the timeout instead of hanging the
// GPU: *err is set and the kernel exits.
struct PeerTable {
    uint32_t* f[8];
};

__global__ void peer_barrier_kernel(PeerTable t, int n, int self, uint32_t target, uint32_t* err,
                                          uint64_t timeout_ns) {
    if (threadIdx.x != 0) return;
    __threadfence_system();
    for (int r = 0; r < n; ++r) atomicAdd_system(t.f[r], 1u);
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    const volatile uint32_t* mine = t.f[self];
    while (static_cast<int32_t>(*mine - target) < 0) {
        uint64_t now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        if (now - t0 > timeout_ns) {
            atomicExch(err, 1u);
            break;
        }
        __nanosleep(256);
    }
    __threadfence_system();
}

}  // namespace
}  // namespace qvk

using namespace qvk;

extern "C" {

int qvk_peer_barrier(qvk_stream_t stream, int32_t n, uint32_t* const* flags_d, int32_t self, uint32_t epoch,
                     uint32_t* err_d) {
    if (n < 1 || n > 8 || !flags_d || self < 0 || self >= n || !err_d)
        QVK_INVALID("peer_barrier: 1..8 ranks, flags and error word required");
    PeerTable t{};
    for (int r = 0; r < n; ++r) {
        if (!flags_d[r]) QVK_INVALID("peer_barrier: null flag pointer");
        t.f[r] = flags_d[r];
    }
    const uint64_t timeout_ns = static_cast<uint64_t>(env_knob("QVK_PEER_BARRIER_TIMEOUT_MS", 20000)) * 1000000ull;
    peer_barrier_kernel<<<1, 32, 0, stream>>>(t, n, self, epoch * static_cast<uint32_t>(n), err_d, timeout_ns);
    QVK_LAUNCH_CHECK();
    return QVK_OK;
}

int qvk_comm_unique_id(void* id_out) {
    if (!id_out) QVK_INVALID("comm: null id buffer");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId id;
    QVK_NCCL(ncclGetUniqueId(&id));
    std::memcpy(id_out, &id, sizeof(id));
    return QVK_OK;
}

int qvk_comm_init(qvk_comm_t* out, int32_t world, int32_t rank, const void* unique_id) {
    if (!out || !unique_id) QVK_INVALID("comm: null argument");
    *out = nullptr;
    if (world < 1 || rank < 0 || rank >= world) QVK_INVALID("comm: rank must be in [0, world)");
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    auto* c = new qvk_comm_st;
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    // world 1 has nothing to overlap: no cap unless QVK_COMM_CTAS is set explicitly (the test hook)
    const int ctas = std::max(0, qvk::env_knob("QVK_COMM_CTAS", world > 1 ? 8 : 0));
    if (ctas > 0) cfg.maxCTAs = ctas;
    ncclResult_t r = ncclCommInitRankConfig(&c->comm, world, id, rank, &cfg);
    bool capped = ctas > 0;
    if (r == ncclInvalidArgument && capped) {  // an NCCL that rejects the cap (same on every rank): uncapped init
        c->comm = nullptr;
        r = ncclCommInitRank(&c->comm, world, id, rank);
        capped = false;
    }
    if (r != ncclSuccess) {
        delete c;
        return nccl_fail(r, "ncclCommInitRankConfig");
    }
    c->rank = rank;
    c->world = world;
    if (capped && ctas < qvk::sm_count() - 2) {  // the all-gather's CTAs get SMs of their own
        int32_t prev = 0;
        qvk_reserve_sms(ctas, &prev);
        c->reserved = ctas;
    }
    *out = c;
    return QVK_OK;
}

int qvk_comm_init_all(qvk_comm_t* comms_out, int32_t n_dev, const int32_t* devices) {
    if (!comms_out || n_dev < 1) QVK_INVALID("comm: null argument");
    std::vector<ncclComm_t> comms(n_dev, nullptr);
    QVK_NCCL(ncclCommInitAll(comms.data(), n_dev, devices));
    for (int i = 0; i < n_dev; ++i) {
        auto* c = new qvk_comm_st;
        c->comm = comms[i];
        c->rank = i;
        c->world = n_dev;
        comms_out[i] = c;
    }
    return QVK_OK;
}

int qvk_comm_wrap(qvk_comm_t* out, void* nccl_comm) {
    if (!out || !nccl_comm) QVK_INVALID("comm: null argument");
    auto* c = new qvk_comm_st;
    c->comm = static_cast<ncclComm_t>(nccl_comm);
    c->owned = false;
    const int rc = fill_rank(c);
    if (rc != QVK_OK) {
        delete c;
        return rc;
    }
    *out = c;
    return QVK_OK;
}

int qvk_comm_rank(qvk_comm_t c, int32_t* rank, int32_t* world) {
    if (!c) QVK_INVALID("comm: null communicator");
    if (rank) *rank = c->rank;
    if (world) *world = c->world;
    return QVK_OK;
}

int qvk_comm_check(qvk_comm_t c) {
    if (!c) QVK_INVALID("comm: null communicator");
    ncclResult_t async = ncclSuccess;
    QVK_NCCL(ncclCommGetAsyncError(c->comm, &async));
    if (async != ncclSuccess && async != ncclInProgress) return nccl_fail(async, "asynchronous collective");
    return QVK_OK;
}

int qvk_comm_destroy(qvk_comm_t c) {
    if (!c) return QVK_OK;
    ncclResult_t r = ncclSuccess;
    if (c->owned && c->comm) {
        r = ncclCommFinalize(c->comm);
        if (r == ncclSuccess) r = ncclCommDestroy(c->comm);
    }
    if (c->reserved) qvk_reserve_sms(0, nullptr);
    delete c;
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommDestroy");
    return QVK_OK;
}

int qvk_comm_group_start(void) {
    QVK_NCCL(ncclGroupStart());
    return QVK_OK;
}

int qvk_comm_group_end(void) {
    QVK_NCCL(ncclGroupEnd());
    return QVK_OK;
}

int qvk_allgather_layer(qvk_stream_t stream, qvk_comm_t c, const int64_t* rank_row_begin, int32_t heads,
                        int32_t width, void* k_cache, void* v_cache, uint64_t* origin) {
    if (!c) QVK_INVALID("comm: null communicator");
    if (!rank_row_begin) QVK_INVALID("allgather: null rank segment table");
    if (heads <= 0 || width <= 0) QVK_INVALID("model config: dimensions must be positive");
    if (!k_cache || !v_cache) QVK_INVALID("allgather: null cache");
    for (int r = 0; r < c->world; ++r)
        if (rank_row_begin[r + 1] < rank_row_begin[r] || rank_row_begin[r] < 0)
            QVK_INVALID("allgather: rank segments must be ascending");
    const size_t row_kv = static_cast<size_t>(heads) * width;  // bf16 elements per cache row of K (or V)
    auto* kc = static_cast<__nv_bfloat16*>(k_cache);
    auto* vc = static_cast<__nv_bfloat16*>(v_cache);
    QVK_NCCL(ncclGroupStart());
    ncclResult_t r_issue = ncclSuccess;
    for (int r = 0; r < c->world && r_issue == ncclSuccess; ++r) {
        const size_t r0 = static_cast<size_t>(rank_row_begin[r]);
        const size_t rows = static_cast<size_t>(rank_row_begin[r + 1]) - r0;
        if (rows == 0) continue;
        // in place: at the root send == recv; everywhere else the segment is received into the same offsets
        r_issue = ncclBroadcast(kc + r0 * row_kv, kc + r0 * row_kv, rows * row_kv * 2, ncclUint8, r, c->comm, stream);
        if (r_issue == ncclSuccess)
            r_issue = ncclBroadcast(vc + r0 * row_kv, vc + r0 * row_kv, rows * row_kv * 2, ncclUint8, r, c->comm,
                                    stream);
        if (r_issue == ncclSuccess && origin)
            r_issue = ncclBroadcast(origin + r0 * heads, origin + r0 * heads, rows * heads, ncclUint64, r, c->comm,
                                    stream);
    }
    const ncclResult_t r_end = ncclGroupEnd();  // the group is always closed; its launch errors surface here
    if (r_issue != ncclSuccess) return nccl_fail(r_issue, "ncclBroadcast");
    if (r_end != ncclSuccess) return nccl_fail(r_end, "ncclGroupEnd");
    return QVK_OK;
}

}  // extern "C"
