// (a4) Per-group causal GQA attention on CTA PAIRS (tcgen05.mma.cta_group::2) — experimental variant of attention.cu
// (QVK_ATTN_2CTA=1).
//
// Why: in attention.cu a CTA ping-pongs two 128-row query tiles and P aliases S in TMEM, so each tile's loop is
// softmax(j) -> PV(j) -> S(j+1) -> softmax(j+1): ~1580 + 1024 cycles per 2048 cycles of tensor work.  Here a CTA pair
// (one cluster on a TPC) owns a 256-row query block; each CTA holds ONE 128-row tile, so its TMEM fits a
// double-buffered S (S(j+1) computes while softmax(j) runs) next to O:
//   TMEM per CTA: S buf 0 [0,128) | S buf 1 [128,256) | O [256,384) | P buf 0 [384,448) | P buf 1 [448,512)
//   MMA order (leader CTA, one thread): S(0) S(1) | S(2) PV(0) | S(3) PV(1) | ... ;  S(j+2) reuses S(j)'s buffer as
//   soon as every softmax warp of both CTAs has read S(j) (s_free), before P(j) exists.  P has its own columns:
//   each softmax warp reads BOTH key halves of S (its own for the exponentials, the other for the row max), so P
//   written over S would race with the other half's read.
// M = 256 pair MMAs: each CTA provides its 128 query rows (A) and HALF of every K tile (64 keys) / V tile (64 head-dim
// columns) as B, so per SM the shared-memory operand + TMA traffic is ~94 B/clk against ~125 for the one-CTA kernel.
// Softmax: 8 warps per CTA, two per TMEM lane quarter splitting the 128 key columns of a row (64 each); the halves
// exchange their row maxima through shared memory each step.  P(j) of key half h is published on p_full[buf][h], so
// PV(j)'s first four k-steps start as soon as both CTAs' first halves are in.  O is rescaled lazily (row max grown by
// > 2^8); since PV(j-1) may still run while softmax(j) does, a rescale first waits for pv_done of PV(j-1).
// Work unit = (group, query head, 256-row block b): 2b+2 K/V steps (the last one fully masked for CTA 0's rows).
#include <cudaTypedefs.h>

#include <cstdlib>

#include "common.cuh"
#include "ptx.cuh"

namespace qvk {
namespace {

constexpr int kD = 128;
constexpr int kRows = 128;                          // query rows per CTA (256 per pair)
constexpr int kKeys = 128;                          // keys per K/V step
constexpr uint32_t kQChunk = kRows * 128;           // 128 rows x 128 B (64 head-dim columns), SW128
constexpr uint32_t kQBytes = 2 * kQChunk;           // 32 KB: the CTA's Q tile
constexpr uint32_t kKChunk = (kKeys / 2) * 128;     // 64 keys x 128 B
constexpr uint32_t kItemBytes = 2 * kKChunk;        // 16 KB: K half (64 keys x 128 d) or V half (128 keys x 64 d)
constexpr int kStages = 8;                          // ring of 16 KB items (K and V halves alternate)
constexpr int kThreads = 512;
constexpr int kEpiWarp0 = 8, kTmaWarp = 12, kMmaWarp = 13;
constexpr int kRegsSoftmax = 168, kRegsEpilogue = 48, kRegsProducer = 96;  // 256*168 + 128*48 + 128*96 <= 64K
constexpr float kRescaleThreshold = 8.0f;

struct Bar2 {
    uint64_t q_full[2], q_empty[2];
    uint64_t kv_full[kStages], kv_empty[kStages];
    uint64_t s_full[2];
    uint64_t s_free[2];     // leader: 2 CTAs x 8 softmax warps have read S(buffer)
    uint64_t p_full[2][2];  // [buffer][key half] — leader: 2 CTAs x 4 softmax warps
    uint64_t pv_done[2];    // PV(k) retired, k = global step (alternating by step parity; multicast commit)
    uint64_t o_done;        // last PV of the unit retired (multicast commit)
    uint64_t o_free;        // leader: 2 CTAs x 128 epilogue threads have read O
    uint64_t l_full, l_free;
    uint32_t tmem_base;
    float row_sum[2][kRows];  // [key half][row]
};
constexpr size_t kSmem = 1024 + 2 * kQBytes + kStages * kItemBytes + sizeof(Bar2);

struct Attn2Params {
    const int64_t* tok_off;
    int n_groups, n_q, n_kv, blocks_max, total_units;
    float scale_log2;
    __nv_bfloat16* o;
};

struct Unit2 {
    int g, hq, hk, b, n, nsteps;
    int64_t tok0;
    bool valid;
};
__device__ __forceinline__ Unit2 decode2(const Attn2Params& p, int u) {
    Unit2 w;
    const int per_block = p.n_groups * p.n_q;
    w.b = p.blocks_max - 1 - u / per_block;  // heaviest blocks first
    const int rem = u % per_block;
    w.g = rem / p.n_q;
    w.hq = rem - w.g * p.n_q;
    w.hk = w.hq / (p.n_q / p.n_kv);
    w.tok0 = __ldg(p.tok_off + w.g);
    w.n = static_cast<int>(__ldg(p.tok_off + w.g + 1) - w.tok0);
    w.valid = w.b * 2 * kRows < w.n;
    const int last_row = min(w.b * 2 * kRows + 2 * kRows - 1, w.n - 1);
    w.nsteps = last_row / kKeys + 1;
    return w;
}

__device__ __forceinline__ uint32_t cta_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t map_rank(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
// Arrive on a barrier of either CTA of the pair (default .release.cta semantics, as CUTLASS's ClusterBarrier: the
// tcgen05.fence::before_thread_sync before it orders this thread's TMEM writes for the MMA issuer).
__device__ __forceinline__ void arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// TMA into this CTA's smem, completing on the LEADER's barrier (cta_group::2 form).
__device__ __forceinline__ void tma3_pair(uint32_t dst, const CUtensorMap* m, uint32_t leader_bar, int c0, int c1,
                                          int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
        "%5}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(leader_bar), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
__device__ __forceinline__ void commit_pair(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            ptx::smem_u32(bar)),
        "h"(static_cast<uint16_t>(3))
        : "memory");
}
__device__ __forceinline__ void mma2_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma2_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a_tmem), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ uint64_t desc_plus(uint64_t d, uint32_t off_bytes) {
    return (d & 0xffffffff00000000ull) | (static_cast<uint32_t>(d) + (off_bytes >> 4));
}

__global__ void __launch_bounds__(kThreads, 1)
    attention2_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                      const __grid_constant__ CUtensorMap tm_v, const Attn2Params p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;                        // [Q buffer] 32 KB
    uint8_t* sR = smem + 2 * kQBytes;          // ring of 16 KB items
    Bar2* bar = reinterpret_cast<Bar2*>(sR + kStages * kItemBytes);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cta_rank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, pairs = gridDim.x >> 1;
    if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&bar->q_full[i], 1);
            ptx::mbar_init(&bar->q_empty[i], 1);
            ptx::mbar_init(&bar->s_full[i], 1);
            ptx::mbar_init(&bar->s_free[i], 2 * 8);
            ptx::mbar_init(&bar->p_full[i][0], 2 * 4);  // one arrival per softmax warp of each CTA
            ptx::mbar_init(&bar->p_full[i][1], 2 * 4);
        }
        for (int s = 0; s < kStages; ++s) {
            ptx::mbar_init(&bar->kv_full[s], 1);
            ptx::mbar_init(&bar->kv_empty[s], 1);
        }
        ptx::mbar_init(&bar->pv_done[0], 1);
        ptx::mbar_init(&bar->pv_done[1], 1);
        ptx::mbar_init(&bar->o_done, 1);
        ptx::mbar_init(&bar->o_free, 2 * 128);
        ptx::mbar_init(&bar->l_full, 256);
        ptx::mbar_init(&bar->l_free, 128);
        ptx::fence_mbar_init();
    }
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         ptx::smem_u32(&bar->tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    ptx::tc_fence_before();
    cluster_sync_all();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = bar->tmem_base;

    if (warp >= kTmaWarp) {
        ptx::setmaxnreg_dec<kRegsProducer>();
        if (warp == kTmaWarp && ptx::elect_one()) {
            // ===================== TMA (both CTAs): this CTA's Q rows and its halves of every K / V tile ===========
            ptx::prefetch_tmap(&tm_q);
            ptx::prefetch_tmap(&tm_k);
            ptx::prefetch_tmap(&tm_v);
            uint32_t item = 0, qi = 0;
            for (int u = pair; u < p.total_units; u += pairs) {
                const Unit2 w = decode2(p, u);
                if (!w.valid) continue;
                const int qb = qi & 1;
                ptx::mbar_wait(&bar->q_empty[qb], ((qi >> 1) & 1) ^ 1);
                if (leader) ptx::mbar_arrive_expect_tx(&bar->q_full[qb], 2 * kQBytes);
                const uint32_t qbar = map_rank(ptx::smem_u32(&bar->q_full[qb]), 0);
                const int qrow = static_cast<int>(w.tok0) + w.b * 2 * kRows + static_cast<int>(rank) * kRows;
                const uint32_t qdst = ptx::smem_u32(sQ + qb * kQBytes);
                tma3_pair(qdst, &tm_q, qbar, 0, w.hq, qrow);
                tma3_pair(qdst + kQChunk, &tm_q, qbar, 64, w.hq, qrow);
                ++qi;
                // order: K0, K1, then per step j: K(j+2), V(j) — the MMA order
                auto push = [&](bool is_v, int j) {
                    const uint32_t st = item % kStages;
                    ptx::mbar_wait(&bar->kv_empty[st], ((item / kStages) & 1) ^ 1);
                    if (leader) ptx::mbar_arrive_expect_tx(&bar->kv_full[st], 2 * kItemBytes);
                    const uint32_t fb = map_rank(ptx::smem_u32(&bar->kv_full[st]), 0);
                    const uint32_t dst = ptx::smem_u32(sR + st * kItemBytes);
                    const int row0 = static_cast<int>(w.tok0) + j * kKeys;
                    if (is_v) {  // all 128 keys, head-dim columns [64 rank, 64 rank + 64)
                        tma3_pair(dst, &tm_v, fb, 64 * static_cast<int>(rank), w.hk, row0);
                    } else {     // keys [64 rank, 64 rank + 64) of the tile, all 128 head-dim columns
                        const int r = row0 + 64 * static_cast<int>(rank);
                        tma3_pair(dst, &tm_k, fb, 0, w.hk, r);
                        tma3_pair(dst + kKChunk, &tm_k, fb, 64, w.hk, r);
                    }
                    ++item;
                };
                push(false, 0);
                if (w.nsteps > 1) push(false, 1);
                for (int j = 0; j < w.nsteps; ++j) {
                    if (j + 2 < w.nsteps) push(false, j + 2);
                    push(true, j);
                }
            }
        } else if (warp == kMmaWarp && leader && ptx::elect_one()) {
            // ===================== MMA issuer (leader CTA, one thread) =====================
            constexpr uint32_t kIdS = ptx::idesc_bf16_f32(2 * kRows, kKeys, false, false);
            constexpr uint32_t kIdPV = ptx::idesc_bf16_f32(2 * kRows, kD, false, true);
            const uint32_t q_base = ptx::smem_u32(sQ), ring = ptx::smem_u32(sR);
            uint32_t item = 0, qi = 0, kstep = 0, o_units = 0;
            auto wait_item = [&]() -> uint32_t {
                const uint32_t st = item % kStages;
                ptx::mbar_wait(&bar->kv_full[st], (item / kStages) & 1);
                ptx::tc_fence_after();
                return st;
            };
            for (int u = pair; u < p.total_units; u += pairs) {
                const Unit2 w = decode2(p, u);
                if (!w.valid) continue;
                const int qb = qi & 1;
                ptx::mbar_wait(&bar->q_full[qb], (qi >> 1) & 1);
                ptx::tc_fence_after();
                const uint32_t qa = q_base + qb * kQBytes;
                const uint64_t dq = ptx::umma_desc_sw128(qa, 16, 1024);
                // S(j) = Q K(j)^T into buffer (kstep + j) & 1
                auto issue_s = [&](int j) {
                    const uint32_t st = wait_item();
                    const uint32_t ka = ring + st * kItemBytes;
                    const uint64_t dk = ptx::umma_desc_sw128(ka, 16, 1024);
                    const uint32_t d = tmem + ((kstep + j) & 1) * 128;
#pragma unroll
                    for (int kk = 0; kk < kD / 16; ++kk) {
                        const uint32_t oq = (kk >> 2) * kQChunk + (kk & 3) * 32;
                        const uint32_t ok = (kk >> 2) * kKChunk + (kk & 3) * 32;
                        mma2_ss(d, desc_plus(dq, oq), desc_plus(dk, ok), kIdS, kk > 0);
                    }
                    commit_pair(&bar->kv_empty[st]);
                    commit_pair(&bar->s_full[(kstep + j) & 1]);
                    ++item;
                    if (j == w.nsteps - 1) commit_pair(&bar->q_empty[qb]);  // the unit's last S issued
                };
                issue_s(0);
                if (w.nsteps > 1) issue_s(1);
                for (int j = 0; j < w.nsteps; ++j) {
                    const uint32_t k = kstep + j, buf = k & 1;
                    if (j + 2 < w.nsteps) {  // S(j+2) reuses S(j)'s buffer as soon as every softmax warp has read it
                        ptx::mbar_wait(&bar->s_free[buf], (k >> 1) & 1);
                        ptx::tc_fence_after();
                        issue_s(j + 2);
                    }
                    const uint32_t st = wait_item();
                    const uint64_t dv = ptx::umma_desc_sw128(ring + st * kItemBytes, kItemBytes, 1024);
                    if (j == 0) ptx::mbar_wait(&bar->o_free, (o_units & 1) ^ 1);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        ptx::mbar_wait(&bar->p_full[buf][h], (k >> 1) & 1);
                        ptx::tc_fence_after();
#pragma unroll
                        for (int kk = 4 * h; kk < 4 * h + 4; ++kk)
                            mma2_ts(tmem + 256, tmem + 384 + buf * 64 + kk * 8, desc_plus(dv, kk * 16 * 128), kIdPV,
                                    (j > 0 || kk > 0) ? 1u : 0u);
                    }
                    commit_pair(&bar->kv_empty[st]);
                    commit_pair(&bar->pv_done[k & 1]);
                    ++item;
                    if (j == w.nsteps - 1) {
                        commit_pair(&bar->o_done);
                        ++o_units;
                    }
                }
                kstep += w.nsteps;
                ++qi;
            }
        }
    } else if (warp >= kEpiWarp0) {
        ptx::setmaxnreg_dec<kRegsEpilogue>();
        // ===================== epilogue: O / l -> bf16 -> HBM =====================
        const int quarter = warp & 3;
        const int r = quarter * 32 + lane;
        const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
        const uint32_t o_free = map_rank(ptx::smem_u32(&bar->o_free), 0);
        uint32_t units = 0;
        for (int u = pair; u < p.total_units; u += pairs) {
            const Unit2 w = decode2(p, u);
            if (!w.valid) continue;
            const uint32_t ph = units & 1;
            ptx::mbar_wait(&bar->l_full, ph);
            const float inv = 1.f / (bar->row_sum[0][r] + bar->row_sum[1][r]);
            ptx::mbar_arrive(&bar->l_free);
            ptx::mbar_wait(&bar->o_done, ph);
            ptx::tc_fence_after();
            const int row = w.b * 2 * kRows + static_cast<int>(rank) * kRows + r;
            __nv_bfloat16* dst = p.o + ((w.tok0 + row) * p.n_q + w.hq) * static_cast<int64_t>(kD);
#pragma unroll
            for (int c = 0; c < kD / 16; ++c) {
                uint32_t o[16];
                QVK_TMEM_LD16(tmem + lane_off + 256 + c * 16, o);
                ptx::tmem_ld_wait();
                if (c == kD / 16 - 1) {
                    ptx::tc_fence_before();
                    arrive_cluster(o_free);
                }
                uint32_t pk[8];
#pragma unroll
                for (int e = 0; e < 8; ++e)
                    pk[e] = ptx::pack_bf16(__uint_as_float(o[2 * e]) * inv, __uint_as_float(o[2 * e + 1]) * inv);
                if (row < w.n) {
                    uint4* d4 = reinterpret_cast<uint4*>(dst + c * 16);
                    d4[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                    d4[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
                }
            }
            ++units;
        }
    } else {
        ptx::setmaxnreg_inc<kRegsSoftmax>();
        // ===================== softmax: warp = (lane quarter, key half) =====================
        const int quarter = warp & 3, h = warp >> 2;
        const int r = quarter * 32 + lane;
        const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
        const float sl2 = p.scale_log2;
        const uint32_t sf0 = map_rank(ptx::smem_u32(&bar->s_free[0]), 0);
        const uint32_t sf1 = map_rank(ptx::smem_u32(&bar->s_free[1]), 0);
        const uint32_t pf0 = map_rank(ptx::smem_u32(&bar->p_full[0][h]), 0);
        const uint32_t pf1 = map_rank(ptx::smem_u32(&bar->p_full[1][h]), 0);
        uint32_t kstep = 0, units = 0;
        for (int u = pair; u < p.total_units; u += pairs) {
            const Unit2 w = decode2(p, u);
            if (!w.valid) continue;
            const int row = w.b * 2 * kRows + static_cast<int>(rank) * kRows + r;  // query row in the group
            float m_ref = -INFINITY, l = 0.f;
            for (int j = 0; j < w.nsteps; ++j) {
                const uint32_t k = kstep + j, buf = k & 1;
                ptx::mbar_wait(&bar->s_full[buf], (k >> 1) & 1);
                ptx::tc_fence_after();
                // this half's 64 columns (kept: its exponentials) and the other half's 64 (row max only), four loads
                // in flight behind one wait — the two halves derive the same row max without a cross-warp exchange
                float x[64], y[64];
                const uint32_t s_col = tmem + lane_off + buf * 128 + h * 64;
                const uint32_t y_col = tmem + lane_off + buf * 128 + (h ^ 1) * 64;
                QVK_TMEM_LD32F(s_col, (x + 0));
                QVK_TMEM_LD32F(s_col + 32, (x + 32));
                QVK_TMEM_LD32F(y_col, (y + 0));
                QVK_TMEM_LD32F(y_col + 32, (y + 32));
                ptx::tmem_ld_wait();
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) arrive_cluster(buf ? sf1 : sf0);  // S(buffer) read: the MMA may overwrite it
                const int key0 = j * kKeys + h * 64, ykey0 = j * kKeys + (h ^ 1) * 64;
                if (key0 + 63 > row) {
#pragma unroll
                    for (int c = 0; c < 64; ++c)
                        if (key0 + c > row) x[c] = -INFINITY;
                }
                if (ykey0 + 63 > row) {
#pragma unroll
                    for (int c = 0; c < 64; ++c)
                        if (ykey0 + c > row) y[c] = -INFINITY;
                }
                float m0 = fmaxf(x[0], y[0]), m1 = fmaxf(x[1], y[1]), m2 = fmaxf(x[2], y[2]), m3 = fmaxf(x[3], y[3]);
#pragma unroll
                for (int c = 4; c < 64; c += 4) {
                    m0 = fmaxf(m0, fmaxf(x[c], y[c]));
                    m1 = fmaxf(m1, fmaxf(x[c + 1], y[c + 1]));
                    m2 = fmaxf(m2, fmaxf(x[c + 2], y[c + 2]));
                    m3 = fmaxf(m3, fmaxf(x[c + 3], y[c + 3]));
                }
                const float mx = fmaxf(fmaxf(m0, m1), fmaxf(m2, m3));
                const float m_new = mx * sl2;
                if (j == 0) {
                    m_ref = m_new;
                } else {
                    const bool need = m_new > m_ref + kRescaleThreshold;
                    if (__any_sync(0xffffffffu, need)) {
                        const float m_upd = need ? m_new : m_ref;
                        const float f = ptx::ex2(m_ref - m_upd);
                        l *= f;
                        m_ref = m_upd;
                        // PV(j-1) (and PV(j-2)) may still accumulate into O: wait for PV(j-1).  S(j) completed and was
                        // issued after PV(j-3), so pv_done[(k-1) & 1]'s previous phase (PV(k-3)) is complete: the
                        // parity wait cannot alias
                        ptx::mbar_wait(&bar->pv_done[(k - 1) & 1], ((k - 1) >> 1) & 1);
                        ptx::tc_fence_after();
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            uint32_t o[16];
                            const uint32_t oc = tmem + lane_off + 256 + h * 64 + c * 16;
                            QVK_TMEM_LD16(oc, o);
                            ptx::tmem_ld_wait();
#pragma unroll
                            for (int e = 0; e < 16; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * f);
                            QVK_TMEM_ST16(oc, o);
                        }
                        ptx::tmem_st_wait();
                    }
                }
                const ptx::f2 sl2x2 = ptx::f2_make(sl2, sl2);
                const float mref_safe = m_ref == -INFINITY ? 0.f : m_ref;  // fully masked rows: exp2(-inf) = 0
                const ptx::f2 negx2 = ptx::f2_make(-mref_safe, -mref_safe);
                ptx::f2 acc0 = ptx::f2_make(0.f, 0.f), acc1 = acc0;
                uint32_t pk[32];
#pragma unroll
                for (int c = 0; c < 32; ++c) {
                    const ptx::f2 y = ptx::f2_fma(ptx::f2_make(x[2 * c], x[2 * c + 1]), sl2x2, negx2);
                    float p0, p1;
                    ptx::f2_split(y, p0, p1);
                    if ((c & 15) < 4) {
                        ptx::ex2_poly2(p0, p1);
                    } else {
                        p0 = ptx::ex2(p0);
                        p1 = ptx::ex2(p1);
                    }
                    if (c & 1) acc1 = ptx::f2_add(acc1, ptx::f2_make(p0, p1));
                    else acc0 = ptx::f2_add(acc0, ptx::f2_make(p0, p1));
                    pk[c] = ptx::pack_bf16(p0, p1);
                }
                // P(k) reuses the P buffer of P(k-2): PV(k-2) must have read it (S(k) was issued before PV(k-2));
                // PV(k-3) retired before S(k) was issued, so pv_done[buf] is at most one phase behind
                if (k >= 2) {
                    ptx::mbar_wait(&bar->pv_done[buf], ((k - 2) >> 1) & 1);
                    ptx::tc_fence_after();
                }
                // P over this half's 32 packed columns of the P buffer (keys 64 h .. 64 h + 63)
                QVK_TMEM_ST16(tmem + lane_off + 384 + buf * 64 + h * 32, pk);
                QVK_TMEM_ST16(tmem + lane_off + 384 + buf * 64 + h * 32 + 16, (pk + 16));
                ptx::tmem_st_wait();
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) arrive_cluster(buf ? pf1 : pf0);  // one (remote) arrival per warp
                float s0, s1, s2, s3;
                ptx::f2_split(acc0, s0, s1);
                ptx::f2_split(acc1, s2, s3);
                l += (s0 + s1) + (s2 + s3);
            }
            if (units) ptx::mbar_wait(&bar->l_free, (units - 1) & 1);
            bar->row_sum[h][r] = l;
            ptx::mbar_arrive(&bar->l_full);
            kstep += w.nsteps;
            ++units;
        }
    }
    ptx::tc_fence_before();
    cluster_sync_all();
    if (warp == kMmaWarp) {
        ptx::tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

bool map3(CUtensorMap* m, const void* base, int heads, int64_t tokens, uint32_t box_rows) {
    const auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(tensor_map_encoder());
    if (!enc) return false;
    cuuint64_t dims[3] = {kD, static_cast<cuuint64_t>(heads), static_cast<cuuint64_t>(tokens)};
    cuuint64_t strides[2] = {kD * 2, static_cast<cuuint64_t>(heads) * kD * 2};
    cuuint32_t box[3] = {64, 1, box_rows};
    cuuint32_t estr[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

int launch_attention2(cudaStream_t stream, const qvk_groups* g, const void* q, const void* k, const void* v, int n_q,
                      int n_kv, float scale, void* o) {
    CUtensorMap mq, mk, mv;
    if (!map3(&mq, q, n_q, g->total_tokens, kRows) || !map3(&mk, k, n_kv, g->total_tokens, kKeys / 2) ||
        !map3(&mv, v, n_kv, g->total_tokens, kKeys)) {
        set_error("attention: cuTensorMapEncodeTiled failed");
        return QVK_E_CUDA;
    }
    Attn2Params prm;
    prm.tok_off = g->tok_off_d;
    prm.n_groups = g->n_groups;
    prm.n_q = n_q;
    prm.n_kv = n_kv;
    prm.blocks_max = static_cast<int>((g->max_tokens + 2 * kRows - 1) / (2 * kRows));
    prm.scale_log2 = scale * 1.4426950408889634f;
    prm.o = static_cast<__nv_bfloat16*>(o);
    const int64_t units = static_cast<int64_t>(prm.blocks_max) * g->n_groups * n_q;
    if (units > 0x7fffffff) QVK_INVALID("attention: too many work units");
    prm.total_units = static_cast<int>(units);
    const int pairs = static_cast<int>(std::min<int64_t>(units, sm_count() / 2));
    QVK_CUDA_CHECK(func_attr(reinterpret_cast<const void*>(attention2_kernel),
                             cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmem)));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(2 * pairs));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    QVK_CUDA_CHECK(cudaLaunchKernelEx(&cfg, attention2_kernel, mq, mk, mv, prm));
    return QVK_OK;
}

}  // namespace qvk
