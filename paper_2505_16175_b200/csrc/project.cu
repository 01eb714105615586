// §8f-1: the QKV projection of a prefill layer as a tcgen05 GEMM with the key-norm score fused into its epilogue.
//
// The reference's stand-in model projects every layer's tokens with two naive fp32 x fp32 -> double GEMMs
// (prefill.cpp:38-54 `matmul`, called by `project`, prefill.cpp:185-190) — >= 97 % of its CPU prefill time
// (SURVEY.md §0.7).  The GQA layer this framework prefills needs Q, K and V:
//     [Q | K | V] (T x (n_q + 2 n_kv) d_h) = X (T x d_model) . W^T,   W: ((n_q + 2 n_kv) d_h) x d_model (row-major)
// bf16 operands, fp32 accumulation in TMEM, bf16 outputs written straight into the three (tokens, heads, d_h) tensors
// the attention / prune kernels consume.  For the columns of K the epilogue also computes the key-norm score of
// every (token, KV head) — -sqrt(sum of squares) of the bf16-rounded row in the reference's sequential double order
// (prefill.cpp:200-212), bit-identical to qvk_score on the stored K — so the prune never re-reads K from HBM.
//
// Kernel: persistent (one CTA per SM), 128 x 256 output tiles (n fastest, so co-resident CTAs share the X row
// block through L2), BK = 64, 4-stage TMA ring (16 KB X + 32 KB W per stage, SWIZZLE_128B, both K-major),
// tcgen05.mma.cta_group::1.kind::f16 M = 128, N = 256, K = 16 issued by one elected thread into one of two
// 256-column TMEM accumulators, so the epilogue of tile i overlaps the main loop of tile i + 1.
// Warps: 0 TMA producer, 1 MMA issuer (+ TMEM owner), 2-5 epilogue (TMEM lane quarter = warp % 4, one output row
// per thread).  Algorithmic FLOPs: 2 T d_model (n_q + 2 n_kv) d_h.
#include <cudaTypedefs.h>

#include <cstdlib>

#include "common.cuh"
#include "ptx.cuh"

namespace qvk {
namespace {

constexpr int kBM = 128, kBN = 256, kBK = 64;
constexpr int kStages = 4;
constexpr uint32_t kABytes = kBM * kBK * 2;   // 16 KB
constexpr uint32_t kBBytes = kBN * kBK * 2;   // 32 KB
constexpr uint32_t kStageBytes = kABytes + kBBytes;
constexpr int kThreads = 192;
constexpr int kTmaWarp = 0, kMmaWarp = 1;

struct ProjParams {
    int64_t m;          // tokens
    int n, k;           // output columns, d_model
    int q_cols, kv_cols, d_h, n_kv;
    __nv_bfloat16 *q, *k_out, *v;
    // fused key-norm (optional)
    double* scores;
    const int64_t* tok_off;
    int n_groups;
    int64_t max_tokens;
};

struct ProjBarriers {
    uint64_t full[kStages], empty[kStages];
    uint64_t acc_full[2], acc_empty[2];
    uint32_t tmem_base;
};

constexpr size_t kSmem = 1024 + kStages * kStageBytes + sizeof(ProjBarriers);

__device__ __forceinline__ uint64_t kdesc(uint32_t tile, int kk) {
    return ptx::umma_desc_sw128(tile + kk * 32, 16, 1024);  // k-step kk: +32 B inside the 128-byte SW128 rows
}

// Epilogue of one 128 x 256 accumulator (thread = output row m, TMEM columns acc .. acc + 255): bf16 into the Q / K /
// V tensors, and for the K heads the key-norm score in the reference's sequential double order (prefill.cpp:207).
// Once the accumulator is read, arrive on acc_empty — in the peer CTA when `remote` (2-SM kernel: the leader's).
__device__ __forceinline__ void store_tile(const ProjParams& p, uint32_t acc, int64_t m, int nt, uint32_t acc_empty,
                                           bool remote) {
    const bool live = m < p.m;
    double ss = 0.0;  // key-norm: running sum of squares of the current K head (reference order)
#pragma unroll 1
    for (int c = 0; c < kBN / 32; ++c) {
        float x[32];
        QVK_TMEM_LD32F(acc + 32 * c, x);
        ptx::tmem_ld_wait();
        if (c == kBN / 32 - 1) {  // accumulator fully read: the MMA warp may reuse it
            ptx::tc_fence_before();
            if (remote)
                asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(acc_empty) : "memory");
            else
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(acc_empty) : "memory");
        }
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) pk[e] = ptx::pack_bf16(x[2 * e], x[2 * e + 1]);
        const int col = nt * kBN + 32 * c;  // global output column of this 32-column chunk
        __nv_bfloat16* dst;
        bool is_k = false;
        int kcol = 0;
        if (col < p.q_cols) {
            dst = p.q + m * p.q_cols + col;
        } else if (col < p.q_cols + p.kv_cols) {
            kcol = col - p.q_cols;
            dst = p.k_out + m * p.kv_cols + kcol;
            is_k = true;
        } else {
            dst = p.v + m * p.kv_cols + (col - p.q_cols - p.kv_cols);
        }
        if (live) {
            uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
            for (int q = 0; q < 4; ++q) d4[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
        }
        if (is_k && p.scores && live) {
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                const double lo = static_cast<double>(__uint_as_float(pk[e] << 16));
                const double hi = static_cast<double>(__uint_as_float(pk[e] & 0xffff0000u));
                ss = __fma_rn(lo, lo, ss);  // squares of bf16 values are exact: rounds like ss + d*d
                ss = __fma_rn(hi, hi, ss);
            }
            if ((kcol + 32) % p.d_h == 0) {  // last chunk of this KV head
                const int h = kcol / p.d_h;
                const int g = find_group_fast(p.tok_off, p.n_groups, m, p.max_tokens);
                const int64_t t0 = __ldg(p.tok_off + g);
                const int64_t n = __ldg(p.tok_off + g + 1) - t0;
                p.scores[p.n_kv * t0 + h * n + (m - t0)] = -__dsqrt_rn(ss);  // key_norm_small
                ss = 0.0;
            }
        }
    }
}

// The same epilogue with coalesced output: each 64-column chunk of the CTA's 128 x 256 accumulator is staged as bf16
// in shared memory (128-byte swizzle, one row per thread) and written by ONE TMA store (16 KB) into the Q, K or V
// tensor it belongs to (64-column chunks never straddle them) — instead of 16-byte per-thread stores, 32 rows per warp
// instruction, which cost two L2 write operations per sector and twice the instructions (ncu vs cuBLAS on the C4
// layer shape).  Two staging buffers: a buffer is rewritten only after its previous store has read it.  Rows past the
// last token are clipped by the TMA.  Named barrier 1 = the 128 epilogue threads.
__device__ __forceinline__ void store_tile_staged(const ProjParams& p, uint32_t acc, int64_t m0, int row, int nt,
                                                  uint32_t acc_empty, bool remote, uint8_t* stage, uint32_t& n_chunk,
                                                  const CUtensorMap* tm_q, const CUtensorMap* tm_k,
                                                  const CUtensorMap* tm_v, bool leader) {
    const int64_t m = m0 + row;
    const bool live = m < p.m;
    double ss = 0.0;
#pragma unroll 1
    for (int c2 = 0; c2 < kBN / 64; ++c2, ++n_chunk) {
        const uint32_t buf = n_chunk & 1;
        if (n_chunk >= 2) {  // this buffer's previous store must have read it
            if (leader) ptx::bulk_wait_group_read<1>();
            ptx::named_bar_sync(1, 128);
        }
        uint8_t* sb = stage + buf * (128 * 128);
        const uint32_t rbase = ptx::smem_u32(sb) + row * 128;
        const int col64 = nt * kBN + 64 * c2;
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
            const int c = 2 * c2 + h;
            float x[32];
            QVK_TMEM_LD32F(acc + 32 * c, x);
            ptx::tmem_ld_wait();
            if (c == kBN / 32 - 1) {  // accumulator fully read: the MMA warp may reuse it
                ptx::tc_fence_before();
                if (remote)
                    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(acc_empty) : "memory");
                else
                    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(acc_empty) : "memory");
            }
            uint32_t pk[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) pk[e] = ptx::pack_bf16(x[2 * e], x[2 * e + 1]);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t u = static_cast<uint32_t>(4 * h + q);  // 16-byte unit of the 128-byte staged row
                ptx::sts128(rbase + ((u ^ (row & 7)) << 4), pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
            }
            const int col = col64 + 32 * h;
            if (p.scores && live && col >= p.q_cols && col < p.q_cols + p.kv_cols) {
                const int kcol = col - p.q_cols;
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    const double lo = static_cast<double>(__uint_as_float(pk[e] << 16));
                    const double hi = static_cast<double>(__uint_as_float(pk[e] & 0xffff0000u));
                    ss = __fma_rn(lo, lo, ss);
                    ss = __fma_rn(hi, hi, ss);
                }
                if ((kcol + 32) % p.d_h == 0) {
                    const int hh = kcol / p.d_h;
                    const int g = find_group_fast(p.tok_off, p.n_groups, m, p.max_tokens);
                    const int64_t t0 = __ldg(p.tok_off + g);
                    const int64_t n = __ldg(p.tok_off + g + 1) - t0;
                    p.scores[p.n_kv * t0 + hh * n + (m - t0)] = -__dsqrt_rn(ss);
                    ss = 0.0;
                }
            }
        }
        ptx::fence_proxy_async_smem();  // generic st.shared -> the TMA engine
        ptx::named_bar_sync(1, 128);
        if (leader) {
            const CUtensorMap* tm;
            int cc;
            if (col64 < p.q_cols) {
                tm = tm_q;
                cc = col64;
            } else if (col64 < p.q_cols + p.kv_cols) {
                tm = tm_k;
                cc = col64 - p.q_cols;
            } else {
                tm = tm_v;
                cc = col64 - p.q_cols - p.kv_cols;
            }
            ptx::tma_store_2d(tm, sb, cc, static_cast<int>(m0));
            ptx::bulk_commit_group();
        }
    }
}

// One staged 64-column chunk of the fast drain below: bf16 words pk[0..31] of output columns col64 .. col64 + 63 of
// row m -> staging buffer (SW128) -> one TMA store; key-norm of the K columns in the reference's order.
__device__ __forceinline__ void emit_chunk(const ProjParams& p, const uint32_t* pk, int64_t m0, int row, int col64,
                                           uint8_t* stage, uint32_t& n_chunk, double& ss,
                                           const CUtensorMap* tm_q, const CUtensorMap* tm_k,
                                           const CUtensorMap* tm_v, bool leader) {
    const int64_t m = m0 + row;
    const uint32_t buf = n_chunk & 1;
    if (n_chunk >= 2) {  // this buffer's previous store must have read it
        if (leader) ptx::bulk_wait_group_read<1>();
        ptx::named_bar_sync(1, 128);
    }
    uint8_t* sb = stage + buf * (128 * 128);
    const uint32_t rbase = ptx::smem_u32(sb) + row * 128;
#pragma unroll
    for (int u = 0; u < 8; ++u)
        ptx::sts128(rbase + ((static_cast<uint32_t>(u) ^ (row & 7)) << 4), pk[4 * u], pk[4 * u + 1], pk[4 * u + 2],
                    pk[4 * u + 3]);
    if (p.scores && m < p.m && col64 >= p.q_cols && col64 < p.q_cols + p.kv_cols) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int kcol = col64 - p.q_cols + 32 * h;
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                const double lo = static_cast<double>(__uint_as_float(pk[16 * h + e] << 16));
                const double hi = static_cast<double>(__uint_as_float(pk[16 * h + e] & 0xffff0000u));
                ss = __fma_rn(lo, lo, ss);
                ss = __fma_rn(hi, hi, ss);
            }
            if ((kcol + 32) % p.d_h == 0) {
                const int hh = kcol / p.d_h;
                const int g = find_group_fast(p.tok_off, p.n_groups, m, p.max_tokens);
                const int64_t t0 = __ldg(p.tok_off + g);
                const int64_t n = __ldg(p.tok_off + g + 1) - t0;
                p.scores[p.n_kv * t0 + hh * n + (m - t0)] = -__dsqrt_rn(ss);
                ss = 0.0;
            }
        }
    }
    ptx::fence_proxy_async_smem();
    ptx::named_bar_sync(1, 128);
    if (leader) {
        const CUtensorMap* tm;
        int cc;
        if (col64 < p.q_cols) {
            tm = tm_q;
            cc = col64;
        } else if (col64 < p.q_cols + p.kv_cols) {
            tm = tm_k;
            cc = col64 - p.q_cols;
        } else {
            tm = tm_v;
            cc = col64 - p.q_cols - p.kv_cols;
        }
        ptx::tma_store_2d(tm, sb, cc, static_cast<int>(m0));
        ptx::bulk_commit_group();
    }
    ++n_chunk;
}

// Fast drain of one 128 x 256 accumulator for the single-buffered wide kernel: the TMEM is read in two batches of
// 128 columns (4 loads, ONE wait each) and released right after the second batch lands — before any conversion or
// store — so the next tile's MMAs wait two TMEM load latencies instead of eight plus the whole store path.
__device__ __forceinline__ void store_tile_fast(const ProjParams& p, uint32_t acc, int64_t m0, int row, int col0,
                                                uint32_t acc_empty, uint8_t* stage, uint32_t& n_chunk,
                                                const CUtensorMap* tm_q, const CUtensorMap* tm_k,
                                                const CUtensorMap* tm_v, bool leader) {
    float x[128];
    uint32_t pa[64];
    QVK_TMEM_LD32F(acc + 0, (x + 0));
    QVK_TMEM_LD32F(acc + 32, (x + 32));
    QVK_TMEM_LD32F(acc + 64, (x + 64));
    QVK_TMEM_LD32F(acc + 96, (x + 96));
    ptx::tmem_ld_wait();
#pragma unroll
    for (int e = 0; e < 64; ++e) pa[e] = ptx::pack_bf16(x[2 * e], x[2 * e + 1]);
    QVK_TMEM_LD32F(acc + 128, (x + 0));
    QVK_TMEM_LD32F(acc + 160, (x + 32));
    QVK_TMEM_LD32F(acc + 192, (x + 64));
    QVK_TMEM_LD32F(acc + 224, (x + 96));
    ptx::tmem_ld_wait();
    ptx::tc_fence_before();
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(acc_empty) : "memory");
    double ss = 0.0;
    emit_chunk(p, pa, m0, row, col0, stage, n_chunk, ss, tm_q, tm_k, tm_v, leader);
    emit_chunk(p, pa + 32, m0, row, col0 + 64, stage, n_chunk, ss, tm_q, tm_k, tm_v, leader);
#pragma unroll
    for (int e = 0; e < 64; ++e) pa[e] = ptx::pack_bf16(x[2 * e], x[2 * e + 1]);
    emit_chunk(p, pa, m0, row, col0 + 128, stage, n_chunk, ss, tm_q, tm_k, tm_v, leader);
    emit_chunk(p, pa + 32, m0, row, col0 + 192, stage, n_chunk, ss, tm_q, tm_k, tm_v, leader);
}

__global__ void __launch_bounds__(kThreads, 1)
    project_qkv_kernel(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_w,
                       const ProjParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    ProjBarriers* bar = reinterpret_cast<ProjBarriers*>(smem + kStages * kStageBytes);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m_tiles = static_cast<int>((p.m + kBM - 1) / kBM);
    const int n_tiles = p.n / kBN;
    const int tiles = m_tiles * n_tiles;
    const int kb_count = p.k / kBK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            ptx::mbar_init(&bar->full[s], 1);
            ptx::mbar_init(&bar->empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&bar->acc_full[b], 1);
            ptx::mbar_init(&bar->acc_empty[b], 128);
        }
        ptx::fence_mbar_init();
    }
    if (warp == kMmaWarp) ptx::tmem_alloc<512>(&bar->tmem_base);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = bar->tmem_base;

    if (warp == kTmaWarp) {
        if (ptx::elect_one()) {
            ptx::prefetch_tmap(&tm_x);
            ptx::prefetch_tmap(&tm_w);
            uint32_t it = 0;
            for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
                const int mt = tile / n_tiles, nt = tile - mt * n_tiles;
                for (int kb = 0; kb < kb_count; ++kb, ++it) {
                    const uint32_t s = it % kStages;
                    ptx::mbar_wait(&bar->empty[s], ((it / kStages) & 1) ^ 1);
                    uint8_t* st = smem + s * kStageBytes;
                    ptx::mbar_arrive_expect_tx(&bar->full[s], kStageBytes);
                    ptx::tma_load_2d(st, &tm_x, &bar->full[s], kb * kBK, mt * kBM);
                    ptx::tma_load_2d(st + kABytes, &tm_w, &bar->full[s], kb * kBK, nt * kBN);
                }
            }
        }
    } else if (warp == kMmaWarp) {
        if (ptx::elect_one()) {
            constexpr uint32_t kId = ptx::idesc_bf16_f32(kBM, kBN, false, false);
            const uint32_t base = ptx::smem_u32(smem);
            uint32_t it = 0, n_acc = 0;
            for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++n_acc) {
                const uint32_t b = n_acc & 1;
                ptx::mbar_wait(&bar->acc_empty[b], ((n_acc >> 1) & 1) ^ 1);
                ptx::tc_fence_after();
                const uint32_t d = tmem + b * kBN;
                for (int kb = 0; kb < kb_count; ++kb, ++it) {
                    const uint32_t s = it % kStages;
                    ptx::mbar_wait(&bar->full[s], (it / kStages) & 1);
                    ptx::tc_fence_after();
                    const uint32_t a_addr = base + s * kStageBytes, b_addr = a_addr + kABytes;
#pragma unroll
                    for (int kk = 0; kk < kBK / 16; ++kk)
                        ptx::mma_ss(d, kdesc(a_addr, kk), kdesc(b_addr, kk), kId, (kb | kk) != 0);
                    ptx::mma_commit(&bar->empty[s]);
                }
                ptx::mma_commit(&bar->acc_full[b]);
            }
        }
    } else {
        // ===================== epilogue: TMEM -> bf16 -> Q / K / V (+ key-norm of the K heads) =====================
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
        uint32_t n_acc = 0;
        for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++n_acc) {
            const int mt = tile / n_tiles, nt = tile - mt * n_tiles;
            const uint32_t b = n_acc & 1;
            ptx::mbar_wait(&bar->acc_full[b], (n_acc >> 1) & 1);
            ptx::tc_fence_after();
            store_tile(p, tmem + lane_off + b * kBN, static_cast<int64_t>(mt) * kBM + row, nt,
                       ptx::smem_u32(&bar->acc_empty[b]), false);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == kMmaWarp) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tmem);
    }
}

// ---------------------------------------------------------------------------------------------------------------------
// 2-SM variant (tcgen05.mma.cta_group::2): a CTA pair (cluster of 2 on one TPC) computes a 256 x 256 output tile with
// M = 256 MMAs issued by the leader CTA.  Each CTA stages its own 128 X rows and HALF of the W tile (128 of the 256
// output columns) per k-block — 32 KB instead of 48 KB per SM per k-block, so L2 -> SMEM traffic and the MMA's
// shared-memory operand reads per FLOP drop by a third, and the ring gets 6 stages.  Each CTA's TMEM holds its 128
// rows x 256 columns of the accumulator (double-buffered), drained by its own epilogue warps.
// Barriers: the TMA of both CTAs signals the leader's full[s] (expect_tx for both halves); the leader's MMA commit
// multicasts empty[s] / acc_full[b] to both CTAs; both CTAs' epilogues arrive on the leader's acc_empty[b].
constexpr int kStages2 = 6;
constexpr uint32_t kBHalf = (kBN / 2) * kBK * 2;       // 16 KB: this CTA's 128 W rows
constexpr uint32_t kStage2 = kABytes + kBHalf;          // 32 KB
struct ProjBarriers2 {
    uint64_t full[kStages2], empty[kStages2];
    uint64_t acc_full[2], acc_empty[2];
    uint32_t tmem_base;
};
constexpr uint32_t kStageOut = 2 * 128 * 128;  // two 128-row x 128-byte bf16 staging buffers of the epilogue
constexpr size_t kSmem2 = 1024 + kStages2 * kStage2 + kStageOut + sizeof(ProjBarriers2);
static_assert(kSmem2 <= 232448, "project: 2-SM kernel shared memory above 227 KB");

__device__ __forceinline__ uint32_t cta_rank_in_cluster() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t map_to_cta(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __launch_bounds__(kThreads, 1)
    project_qkv_2sm_kernel(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_w,
                           const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                           const __grid_constant__ CUtensorMap tm_v,
                           const ProjParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* stage_out = smem + kStages2 * kStage2;  // 1024-aligned (SWIZZLE_128B staging of the epilogue)
    ProjBarriers2* bar = reinterpret_cast<ProjBarriers2*>(stage_out + kStageOut);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cta_rank_in_cluster();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, pairs = gridDim.x >> 1;
    const int m_tiles = static_cast<int>((p.m + 2 * kBM - 1) / (2 * kBM));
    const int n_tiles = p.n / kBN;
    const int tiles = m_tiles * n_tiles;
    const int kb_count = p.k / kBK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages2; ++s) {
            ptx::mbar_init(&bar->full[s], 1);   // the leader's expect_tx arrival (tx: both CTAs' TMA)
            ptx::mbar_init(&bar->empty[s], 1);  // the leader's multicast MMA commit
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&bar->acc_full[b], 1);
            ptx::mbar_init(&bar->acc_empty[b], 2 * 128);  // both CTAs' epilogue threads (leader's copy is used)
        }
        ptx::fence_mbar_init();
    }
    if (warp == kMmaWarp) {  // one warp of EACH CTA of the pair allocates collectively
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         ptx::smem_u32(&bar->tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    ptx::tc_fence_before();
    cluster_sync_all();  // barriers of both CTAs initialised, TMEM allocated
    __syncthreads();     // (also orders the allocator's smem write of tmem_base for the CTA-local readers)
    ptx::tc_fence_after();
    const uint32_t tmem = bar->tmem_base;

    if (warp == kTmaWarp) {
        if (ptx::elect_one()) {
            ptx::prefetch_tmap(&tm_x);
            ptx::prefetch_tmap(&tm_w);
            uint32_t it = 0;
            for (int tile = pair; tile < tiles; tile += pairs) {
                const int mt = tile / n_tiles, nt = tile - mt * n_tiles;
                for (int kb = 0; kb < kb_count; ++kb, ++it) {
                    const uint32_t s = it % kStages2;
                    ptx::mbar_wait(&bar->empty[s], ((it / kStages2) & 1) ^ 1);
                    uint8_t* st = smem + s * kStage2;
                    if (leader) ptx::mbar_arrive_expect_tx(&bar->full[s], 2 * kStage2);
                    const uint32_t fb = map_to_cta(ptx::smem_u32(&bar->full[s]), 0);  // the leader's full[s]
                    asm volatile(
                        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
                        "[%0], [%1, {%3, %4}], [%2];" ::"r"(ptx::smem_u32(st)),
                        "l"(reinterpret_cast<uint64_t>(&tm_x)), "r"(fb), "r"(kb * kBK),
                        "r"(mt * 2 * kBM + static_cast<int>(rank) * kBM)
                        : "memory");
                    asm volatile(
                        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
                        "[%0], [%1, {%3, %4}], [%2];" ::"r"(ptx::smem_u32(st + kABytes)),
                        "l"(reinterpret_cast<uint64_t>(&tm_w)), "r"(fb), "r"(kb * kBK),
                        "r"(nt * kBN + static_cast<int>(rank) * (kBN / 2))
                        : "memory");
                }
            }
        }
    } else if (warp == kMmaWarp) {
        if (leader && ptx::elect_one()) {
            constexpr uint32_t kId = ptx::idesc_bf16_f32(2 * kBM, kBN, false, false);
            const uint32_t base = ptx::smem_u32(smem);
            uint32_t it = 0, n_acc = 0;
            for (int tile = pair; tile < tiles; tile += pairs, ++n_acc) {
                const uint32_t b = n_acc & 1;
                ptx::mbar_wait(&bar->acc_empty[b], ((n_acc >> 1) & 1) ^ 1);
                ptx::tc_fence_after();
                const uint32_t d = tmem + b * kBN;
                for (int kb = 0; kb < kb_count; ++kb, ++it) {
                    const uint32_t s = it % kStages2;
                    ptx::mbar_wait(&bar->full[s], (it / kStages2) & 1);
                    ptx::tc_fence_after();
                    const uint32_t a_addr = base + s * kStage2, b_addr = a_addr + kABytes;
#pragma unroll
                    for (int kk = 0; kk < kBK / 16; ++kk) {
                        const uint64_t da = kdesc(a_addr, kk), db = kdesc(b_addr, kk);
                        const uint32_t acc = (kb | kk) != 0;
                        asm volatile(
                            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                            "l"(da), "l"(db), "r"(kId), "r"(acc));
                    }
                    asm volatile(
                        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], "
                        "%1;" ::"r"(ptx::smem_u32(&bar->empty[s])),
                        "h"(static_cast<uint16_t>(3))
                        : "memory");
                }
                asm volatile(
                    "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], "
                    "%1;" ::"r"(ptx::smem_u32(&bar->acc_full[b])),
                    "h"(static_cast<uint16_t>(3))
                    : "memory");
            }
        }
    } else {
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
        uint32_t n_acc = 0, n_chunk = 0;
        const bool out_leader = warp == 2 && lane == 0;  // issues the epilogue's TMA stores
        if (out_leader) {
            ptx::prefetch_tmap(&tm_q);
            ptx::prefetch_tmap(&tm_k);
            ptx::prefetch_tmap(&tm_v);
        }
        for (int tile = pair; tile < tiles; tile += pairs, ++n_acc) {
            const int mt = tile / n_tiles, nt = tile - mt * n_tiles;
            const uint32_t b = n_acc & 1;
            ptx::mbar_wait(&bar->acc_full[b], (n_acc >> 1) & 1);
            ptx::tc_fence_after();
            const int64_t m0 = static_cast<int64_t>(mt) * 2 * kBM + static_cast<int64_t>(rank) * kBM;
            store_tile_staged(p, tmem + lane_off + b * kBN, m0, row, nt,
                              map_to_cta(ptx::smem_u32(&bar->acc_empty[b]), 0), true, stage_out, n_chunk, &tm_q,
                              &tm_k, &tm_v, out_leader);
        }
        if (out_leader) ptx::bulk_wait_group<0>();  // every output store complete before the CTA retires
    }
    ptx::tc_fence_before();
    cluster_sync_all();  // both CTAs done with TMEM (and with the leader's barriers)
    if (warp == kMmaWarp) {
        ptx::tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

// ---------------------------------------------------------------------------------------------------------------------
// Wide 2-SM variant: a CTA pair computes a 256 x 512 output tile as two M = 256, N = 256 MMAs per k-step ("sub-tiles"
// 0 and 1), so every k-block's X rows are staged once for 512 output columns instead of 256 — L2 -> SMEM operand
// traffic per FLOP drops by a quarter (X 16 KB + W 2 x 16 KB per CTA per k-block for 2 x 256 x 256 x 64 MACs).
// Each CTA's whole TMEM (512 columns) is the accumulator: sub-tile j in columns [256 j, 256 j + 256), single-buffered,
// one acc_full / acc_empty barrier per sub-tile.  To overlap the drain anyway, the MMA issuer runs sub-tile 1 kSkew
// k-blocks BEHIND sub-tile 0 (a stage is released by sub-tile 1's commit): sub-tile 0 of a tile completes early and
// is drained (store_tile_fast: released after two TMEM load batches) while the tensor pipe finishes sub-tile 1.
constexpr int kStagesW = 4;
constexpr uint32_t kStageW = kABytes + 2 * kBHalf;  // 48 KB: X 128 rows + W 2 x 128 rows
struct ProjBarriersW {
    uint64_t full[kStagesW], empty[kStagesW];
    uint64_t acc_full[2], acc_empty[2];  // per sub-tile
    uint32_t tmem_base;
};
constexpr size_t kSmemW = 1024 + kStagesW * kStageW + kStageOut + sizeof(ProjBarriersW);
static_assert(kSmemW <= 232448, "project: wide 2-SM kernel shared memory above 227 KB");

__device__ __forceinline__ void mma2_kblock(uint32_t d, uint32_t a_addr, uint32_t b_addr, uint32_t id, bool first) {
#pragma unroll
    for (int kk = 0; kk < kBK / 16; ++kk) {
        const uint64_t da = kdesc(a_addr, kk), db = kdesc(b_addr, kk);
        const uint32_t acc = (!first || kk != 0) ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
            "l"(da), "l"(db), "r"(id), "r"(acc));
    }
}
__device__ __forceinline__ void commit2_multicast(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            ptx::smem_u32(bar)),
        "h"(static_cast<uint16_t>(3))
        : "memory");
}

template <int kSkew>
__global__ void __launch_bounds__(kThreads, 1)
    project_qkv_2sm_wide_kernel(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_w,
                                const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                                const __grid_constant__ CUtensorMap tm_v, const ProjParams p) {
    static_assert(kStagesW >= kSkew + 2, "wide projection: the ring must hold the skew plus one stage in flight");
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* stage_out = smem + kStagesW * kStageW;
    ProjBarriersW* bar = reinterpret_cast<ProjBarriersW*>(stage_out + kStageOut);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cta_rank_in_cluster();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, pairs = gridDim.x >> 1;
    constexpr int kBNW = 2 * kBN;
    const int m_tiles = static_cast<int>((p.m + 2 * kBM - 1) / (2 * kBM));
    const int n_tiles = p.n / kBNW;
    const int tiles = m_tiles * n_tiles;
    const int kb_count = p.k / kBK;
    const int my_tiles = pair < tiles ? (tiles - pair + pairs - 1) / pairs : 0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStagesW; ++s) {
            ptx::mbar_init(&bar->full[s], 1);
            ptx::mbar_init(&bar->empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&bar->acc_full[b], 1);
            ptx::mbar_init(&bar->acc_empty[b], 2 * 128);
        }
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

    if (warp == kTmaWarp) {
        if (ptx::elect_one()) {
            ptx::prefetch_tmap(&tm_x);
            ptx::prefetch_tmap(&tm_w);
            uint32_t it = 0;
            for (int tile = pair; tile < tiles; tile += pairs) {
                const int mt = tile / n_tiles, nt = tile - mt * n_tiles;
                for (int kb = 0; kb < kb_count; ++kb, ++it) {
                    const uint32_t s = it % kStagesW;
                    ptx::mbar_wait(&bar->empty[s], ((it / kStagesW) & 1) ^ 1);
                    const uint32_t st = ptx::smem_u32(smem + s * kStageW);
                    if (leader) ptx::mbar_arrive_expect_tx(&bar->full[s], 2 * kStageW);
                    const uint32_t fb = map_to_cta(ptx::smem_u32(&bar->full[s]), 0);  // the leader's full[s]
                    asm volatile(
                        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
                        "[%0], [%1, {%3, %4}], [%2];" ::"r"(st),
                        "l"(reinterpret_cast<uint64_t>(&tm_x)), "r"(fb), "r"(kb * kBK),
                        "r"(mt * 2 * kBM + static_cast<int>(rank) * kBM)
                        : "memory");
#pragma unroll
                    for (int j = 0; j < 2; ++j)
                        asm volatile(
                            "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
                            "[%0], [%1, {%3, %4}], [%2];" ::"r"(st + kABytes + j * kBHalf),
                            "l"(reinterpret_cast<uint64_t>(&tm_w)), "r"(fb), "r"(kb * kBK),
                            "r"(nt * kBNW + j * kBN + static_cast<int>(rank) * (kBN / 2))
                            : "memory");
                }
            }
        }
    } else if (warp == kMmaWarp) {
        if (leader && ptx::elect_one()) {
            constexpr uint32_t kId = ptx::idesc_bf16_f32(2 * kBM, kBN, false, false);
            const uint32_t base = ptx::smem_u32(smem);
            const int total = my_tiles * kb_count;
            // step i: sub-tile 1 of k-block i - kSkew (releases its stage), then sub-tile 0 of k-block i
            for (int i = 0; i < total + kSkew; ++i) {
                const int j = i - kSkew;
                if (j >= 0) {
                    const int tj = j / kb_count, kbj = j - tj * kb_count;
                    const uint32_t s = static_cast<uint32_t>(j) % kStagesW;
                    if (kbj == 0) {
                        ptx::mbar_wait(&bar->acc_empty[1], (tj & 1) ^ 1);
                        ptx::tc_fence_after();
                    }
                    const uint32_t a_addr = base + s * kStageW;
                    mma2_kblock(tmem + kBN, a_addr, a_addr + kABytes + kBHalf, kId, kbj == 0);
                    commit2_multicast(&bar->empty[s]);
                    if (kbj == kb_count - 1) commit2_multicast(&bar->acc_full[1]);
                }
                if (i < total) {
                    const int ti = i / kb_count, kb = i - ti * kb_count;
                    const uint32_t s = static_cast<uint32_t>(i) % kStagesW;
                    if (kb == 0) {
                        ptx::mbar_wait(&bar->acc_empty[0], (ti & 1) ^ 1);
                        ptx::tc_fence_after();
                    }
                    ptx::mbar_wait(&bar->full[s], (static_cast<uint32_t>(i) / kStagesW) & 1);
                    ptx::tc_fence_after();
                    const uint32_t a_addr = base + s * kStageW;
                    mma2_kblock(tmem, a_addr, a_addr + kABytes, kId, kb == 0);
                    if (kb == kb_count - 1) commit2_multicast(&bar->acc_full[0]);
                }
            }
        }
    } else {
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
        uint32_t n_acc = 0, n_chunk = 0;
        const bool out_leader = warp == 2 && lane == 0;
        if (out_leader) {
            ptx::prefetch_tmap(&tm_q);
            ptx::prefetch_tmap(&tm_k);
            ptx::prefetch_tmap(&tm_v);
        }
        for (int tile = pair; tile < tiles; tile += pairs, ++n_acc) {
            const int mt = tile / n_tiles, nt = tile - mt * n_tiles;
            const int64_t m0 = static_cast<int64_t>(mt) * 2 * kBM + static_cast<int64_t>(rank) * kBM;
#pragma unroll 1
            for (int sub = 0; sub < 2; ++sub) {
                ptx::mbar_wait(&bar->acc_full[sub], n_acc & 1);
                ptx::tc_fence_after();
                store_tile_fast(p, tmem + lane_off + sub * kBN, m0, row, nt * kBNW + sub * kBN,
                                map_to_cta(ptx::smem_u32(&bar->acc_empty[sub]), 0), stage_out, n_chunk, &tm_q,
                                &tm_k, &tm_v, out_leader);
            }
        }
        if (out_leader) ptx::bulk_wait_group<0>();
    }
    ptx::tc_fence_before();
    cluster_sync_all();
    if (warp == kMmaWarp) {
        ptx::tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

bool make_map_2d(CUtensorMap* m, const void* base, int64_t rows, int cols, int box_rows) {
    const auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(tensor_map_encoder());
    if (!enc) return false;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 2};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), static_cast<cuuint32_t>(box_rows)};
    cuuint32_t estr[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_map_out(CUtensorMap* m, const void* base, int64_t rows, int cols) {
    const auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(tensor_map_encoder());
    if (!enc) return false;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 2};
    cuuint32_t box[2] = {64, static_cast<cuuint32_t>(kBM)};
    cuuint32_t estr[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

int launch_project_qkv(cudaStream_t stream, const void* x, int64_t tokens, int d_model, const void* w, int n_q,
                       int n_kv, int d_h, void* q, void* k, void* v, const qvk_groups* g, double* scores) {
    const int n = (n_q + 2 * n_kv) * d_h;
    if (tokens < 0 || d_model <= 0 || n_q <= 0 || n_kv <= 0 || d_h <= 0)
        QVK_INVALID("model config: dimensions must be positive");
    if (d_h % 32 != 0 || kBN % d_h != 0 || d_model % kBK != 0 || n % kBN != 0) {
        set_error("project: needs d_h % 32 == 0, d_model % 64 == 0 and (n_q + 2 n_kv) d_h % 256 == 0");
        return QVK_E_UNSUPPORTED;
    }
    if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(q) |
         reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v)) & 15)
        QVK_INVALID("project: tensors must be 16-byte aligned");
    if (scores && (!g || g->total_tokens != tokens)) QVK_INVALID("project: scores need the token groups");
    if (tokens == 0) return QVK_OK;
    CUtensorMap mx, mw;
    if (!make_map_2d(&mx, x, tokens, d_model, kBM) || !make_map_2d(&mw, w, n, d_model, kBN)) {
        set_error("project: cuTensorMapEncodeTiled failed");
        return QVK_E_CUDA;
    }
    ProjParams p;
    p.m = tokens;
    p.n = n;
    p.k = d_model;
    p.q_cols = n_q * d_h;
    p.kv_cols = n_kv * d_h;
    p.d_h = d_h;
    p.n_kv = n_kv;
    p.q = static_cast<__nv_bfloat16*>(q);
    p.k_out = static_cast<__nv_bfloat16*>(k);
    p.v = static_cast<__nv_bfloat16*>(v);
    p.scores = scores;
    p.tok_off = g ? g->tok_off_d : nullptr;
    p.n_groups = g ? g->n_groups : 0;
    p.max_tokens = g ? g->max_tokens : 0;
    QVK_CUDA_CHECK(func_attr(reinterpret_cast<const void*>(project_qkv_kernel),
                             cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmem)));
    const int sms = grid_sms();
    static const int two_sm = env_knob("QVK_PROJ_2SM", 1) != 0;  // tuning knob QVK_PROJ_2SM = 0 | 1
    if (two_sm) {
        CUtensorMap mw2;  // W boxes of 128 rows: each CTA of the pair stages half of the 256-column tile
        if (!make_map_2d(&mw2, w, n, d_model, kBN / 2)) {
            set_error("project: cuTensorMapEncodeTiled failed");
            return QVK_E_CUDA;
        }
        // QVK_PROJ_WIDE = 0 (256 x 256 pair tiles) | 1 | 2 (256 x 512 pair tiles, sub-tile skew 1 or 2 k-blocks)
        static const int wide_knob = env_knob("QVK_PROJ_WIDE", 0);
        const bool wide = wide_knob != 0 && n % (2 * kBN) == 0;
        const void* kfn = !wide ? reinterpret_cast<const void*>(project_qkv_2sm_kernel)
                          : wide_knob == 2 ? reinterpret_cast<const void*>(project_qkv_2sm_wide_kernel<2>)
                                           : reinterpret_cast<const void*>(project_qkv_2sm_wide_kernel<1>);
        const size_t smem_bytes = wide ? kSmemW : kSmem2;
        QVK_CUDA_CHECK(func_attr(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_bytes)));
        const int64_t tiles2 = ((tokens + 2 * kBM - 1) / (2 * kBM)) * (n / (wide ? 2 * kBN : kBN));
        if (tiles2 > 0x7fffffff) QVK_INVALID("project: too many tiles");
        const unsigned pairs = static_cast<unsigned>(std::min<int64_t>(tiles2, sms / 2));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(2 * pairs);
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = smem_bytes;
        cfg.stream = stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        CUtensorMap mq, mk, mv;  // outputs: boxes of 64 columns x 128 rows (one staged chunk)
        if (!make_map_out(&mq, q, tokens, p.q_cols) || !make_map_out(&mk, k, tokens, p.kv_cols) ||
            !make_map_out(&mv, v, tokens, p.kv_cols)) {
            set_error("project: cuTensorMapEncodeTiled failed");
            return QVK_E_CUDA;
        }
        if (wide && wide_knob == 2)
            QVK_CUDA_CHECK(cudaLaunchKernelEx(&cfg, project_qkv_2sm_wide_kernel<2>, mx, mw2, mq, mk, mv, p));
        else if (wide)
            QVK_CUDA_CHECK(cudaLaunchKernelEx(&cfg, project_qkv_2sm_wide_kernel<1>, mx, mw2, mq, mk, mv, p));
        else
            QVK_CUDA_CHECK(cudaLaunchKernelEx(&cfg, project_qkv_2sm_kernel, mx, mw2, mq, mk, mv, p));
        return QVK_OK;
    }
    const int64_t tiles = ((tokens + kBM - 1) / kBM) * (n / kBN);
    if (tiles > 0x7fffffff) QVK_INVALID("project: too many tiles");
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(tiles, sms));
    project_qkv_kernel<<<grid, kThreads, kSmem, stream>>>(mx, mw, p);
    QVK_LAUNCH_CHECK();
    return QVK_OK;
}

}  // namespace qvk
