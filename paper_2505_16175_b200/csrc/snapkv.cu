// (a7) SnapKV observation-window scores (north star (3); no reference code — DESIGN.md §3.3 states the definition):
//   window rows r in [N - W, N), W = min(window, N); for KV head h and each of its n_q/n_kv query heads:
//   s[h, j] += causal softmax_j(scale * q_r . k_j)  (j <= r);  optional average pooling (odd width, zero padded).
// Two passes over K per (group, head): (1) per window row max/sum of the causal logits, (2) per key the sum of the
// normalised probabilities.  fp32 FMA on CUDA cores; HBM reads of K are the algorithmic bytes
// (N * d * 2 + W * n_q * d * 2 read, N * n_kv * 8 written per group).
#include <cudaTypedefs.h>

#include <cstdlib>

#include "common.cuh"
#include "ptx.cuh"

namespace qvk {
namespace {

constexpr int kD = 128;
constexpr int kRows = 32;  // window rows per CTA pass (stats kernel)
constexpr int kKeys = 32;  // keys per chunk (stats kernel)

__device__ __forceinline__ float bf(const __nv_bfloat16 x) { return __bfloat162float(x); }

// grid (G, n_q): row statistics (max, sum of exp2) of the window rows of query head hq.
__global__ void __launch_bounds__(256) snap_stats_kernel(const __nv_bfloat16* __restrict__ q,
                                                         const __nv_bfloat16* __restrict__ k,
                                                         const int64_t* __restrict__ tok_off, int n_q, int n_kv,
                                                         int window, float sl2, float2* __restrict__ stats) {
    __shared__ float qs[kRows][kD + 1];
    __shared__ float ks[kKeys][kD + 1];
    const int g = blockIdx.x, hq = blockIdx.y, hk = hq / (n_q / n_kv);
    const int64_t t0 = tok_off[g];
    const int n = static_cast<int>(tok_off[g + 1] - t0);
    const int w = min(window, n);
    const int rl = threadIdx.x >> 3, kl = threadIdx.x & 7;  // 32 rows x 8 key lanes
    for (int rb = 0; rb < w; rb += kRows) {
        __syncthreads();
        for (int e = threadIdx.x; e < kRows * kD; e += 256) {
            const int r = e / kD, c = e % kD;
            const int pos = n - w + rb + r;
            qs[r][c] = (rb + r < w) ? bf(q[((t0 + pos) * n_q + hq) * kD + c]) : 0.f;
        }
        const int my_pos = n - w + rb + rl;  // causal limit of this thread's row
        float m = -INFINITY, l = 0.f;
        const int last_key = min(n, n - w + rb + kRows);  // keys beyond every row's position are never needed
        for (int j0 = 0; j0 < last_key; j0 += kKeys) {
            __syncthreads();
            for (int e = threadIdx.x; e < kKeys * kD; e += 256) {
                const int jj = e / kD, c = e % kD;
                ks[jj][c] = (j0 + jj < n) ? bf(k[((t0 + j0 + jj) * n_kv + hk) * kD + c]) : 0.f;
            }
            __syncthreads();
            if (rb + rl < w) {
                for (int jj = kl; jj < kKeys; jj += 8) {
                    const int j = j0 + jj;
                    if (j > my_pos) break;
                    float dot = 0.f;
#pragma unroll 16
                    for (int c = 0; c < kD; ++c) dot = fmaf(qs[rl][c], ks[jj][c], dot);
                    const float x = dot * sl2;
                    if (x > m) {
                        l = l * exp2f(m - x) + 1.f;
                        m = x;
                    } else {
                        l += exp2f(x - m);
                    }
                }
            }
        }
        // merge the 8 key lanes of each row
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
            const float l2 = __shfl_xor_sync(0xffffffffu, l, o);
            const float mm = fmaxf(m, m2);
            l = (m == -INFINITY ? 0.f : l * exp2f(m - mm)) + (m2 == -INFINITY ? 0.f : l2 * exp2f(m2 - mm));
            m = mm;
        }
        if (kl == 0 && rb + rl < w) stats[(static_cast<int64_t>(g) * n_q + hq) * window + rb + rl] = make_float2(m, l);
    }
}

// grid (G, n_kv, ceil(max_n / 128)): one thread per key j sums the normalised probabilities over window rows.
__global__ void __launch_bounds__(128) snap_colsum_kernel(const __nv_bfloat16* __restrict__ q,
                                                          const __nv_bfloat16* __restrict__ k,
                                                          const int64_t* __restrict__ tok_off, int n_q, int n_kv,
                                                          int window, float sl2, const float2* __restrict__ stats,
                                                          float* __restrict__ out) {
    __shared__ float qs[kD];
    const int g = blockIdx.x, hk = blockIdx.y;
    const int64_t t0 = tok_off[g];
    const int n = static_cast<int>(tok_off[g + 1] - t0);
    const int j = blockIdx.z * 128 + threadIdx.x;
    if (blockIdx.z * 128 >= n) return;
    const int w = min(window, n);
    const int ratio = n_q / n_kv;
    float kr[kD];
    if (j < n) {
#pragma unroll
        for (int c = 0; c < kD; ++c) kr[c] = bf(k[((t0 + j) * n_kv + hk) * kD + c]);
    }
    float acc = 0.f;
    for (int gq = 0; gq < ratio; ++gq) {
        const int hq = hk * ratio + gq;
        for (int r = 0; r < w; ++r) {
            const int pos = n - w + r;
            __syncthreads();
            qs[threadIdx.x] = bf(q[((t0 + pos) * n_q + hq) * kD + threadIdx.x]);
            __syncthreads();
            if (j < n && j <= pos) {
                float dot = 0.f;
#pragma unroll
                for (int c = 0; c < kD; ++c) dot = fmaf(qs[c], kr[c], dot);
                const float2 st = stats[(static_cast<int64_t>(g) * n_q + hq) * window + r];
                acc += exp2f(dot * sl2 - st.x) / st.y;
            }
        }
    }
    if (j < n) out[n_kv * t0 + static_cast<int64_t>(hk) * n + j] = acc;
}

// Average pooling (odd width, zero padded, divided by width) per (group, head) segment, float -> double scores.
__global__ void snap_pool_kernel(const float* __restrict__ raw, const int64_t* __restrict__ tok_off, int n_groups,
                                 int heads, int64_t total, int pool, double* __restrict__ out) {
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        // e indexes the (group, head, token) layout: group g spans [heads*tok_off[g], heads*tok_off[g+1]).
        int lo = 0, hi = n_groups - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (heads * __ldg(tok_off + mid) <= e) lo = mid; else hi = mid - 1;
        }
        const int g = lo;
        const int64_t t0 = __ldg(tok_off + g);
        const int64_t n = __ldg(tok_off + g + 1) - t0;
        const int64_t seg0 = heads * t0 + ((e - heads * t0) / n) * n;
        const int64_t j = e - seg0;
        float a = 0.f;
        if (pool <= 1) {
            a = raw[e];
            out[e] = static_cast<double>(a);
            continue;
        }
        const int half = pool / 2;
        for (int u = -half; u <= half; ++u)
            if (j + u >= 0 && j + u < n) a += raw[seg0 + j + u];
        out[e] = static_cast<double>(a) / pool;
    }
}

// ---------------------------------------------------------------------------------------------------------------
// tcgen05 path (d_h = 128, gq = n_q / n_kv <= 256): the gq * W window query rows of a KV head (gq heads x W rows,
// 224 at the default W = 32, GQA 7) are one smem operand of <= 256 rows; larger windows are cut into nb blocks of
// wb window rows (gq * wb <= 256) that the item's CTA runs one after another, each block's per-key sums added to
// the earlier blocks'.  Both passes run on the tensor pipe and the exponentials on the CUDA cores.
//   pass 1  S  = Q_obs K_t^T  (M = 128 window rows per MMA, two M-tiles; N = 128 keys): row max / sum, online over
//           key tiles — thread-local (thread = TMEM lane = window row);
//   pass 2  S' = K_t Q_obs^T  (M = 128 keys, N = ceil32(gq W) window rows): per-key sum of the normalised
//           probabilities — again thread-local (thread = key), so no cross-thread column reduction is needed.
// Work item = (group, KV head), persistent over items.  576 threads: warps 0-15 = four compute sets of four warps
// (one warp per TMEM lane quarter each; four warps per SM sub-partition keep the MUFU busy — two were ~50 % idle on
// latency), warp 16 TMA, warp 17 MMA.  Pass 1: set s takes M-tile s & 1 (window rows 0-127 / 128-255) and key
// columns 64 (s >> 1) .. +63 of every key tile, each keeping its own running (max, sum) per row, merged once per
// item; pass 2: set s takes window columns 64 s .. 64 s + 63, the four partial per-key sums combined through smem.
// TMEM: two accumulator buffers of 256 columns (pass 1: S_A | S_B, pass 2: S' of <= 256 columns), so the MMAs of
// key tile t + 1 run while the compute warps work on tile t (single-buffered, every tile waited for the slowest warp's
// release, then the MMA issue and execution: ~2400 cycles per tile against ~1900 of math, tools/snap_trace.cu).
// Algorithmic bytes per (group, layer): K read once from HBM (pass 2 re-reads it from L2) + the window Q rows +
// n_kv * N * 8 score bytes.
constexpr int kSnapStages = 3;
constexpr uint32_t kSnapChunk = 128 * 128;          // 128 rows x 128 B (one SW128 chunk of a key tile)
constexpr uint32_t kSnapKTile = 2 * kSnapChunk;      // 128 keys x 128 d bf16
constexpr uint32_t kSnapQChunk = 256 * 128;          // window-row operand: up to 256 rows x 128 B per d-chunk
#ifndef QVK_SNAP_POLY8
#define QVK_SNAP_POLY8 2  // exponential pairs of every 8 computed on the FMA pipe instead of the MUFU (0..8)
#endif
constexpr int kSnapThreads = 576;
constexpr int kSnapCompute = 512;  // compute threads (warps 0-15)
constexpr int kSnapTmaWarp = 16, kSnapMmaWarp = 17;

// Exponential pair pi (two adjacent columns) goes to the FMA pipe (ptx::ex2_poly2) for QVK_SNAP_POLY8 of every 8
// pairs, spread evenly (e.g. 3 -> pairs 0, 3, 6 of each 8).  The MUFU does 16 ex2/clk/SM; the polynomial costs
// 8 FMA-pipe cycles per element per SM sub-partition, so the pipes balance near 3/8 with the other per-element work.
__host__ __device__ constexpr bool kSnapPoly(int pi) { return (pi * QVK_SNAP_POLY8) % 8 < QVK_SNAP_POLY8; }
struct SnapShared {
    uint64_t q_full, q_empty, acc_full[2], acc_empty[2];
    uint64_t kv_full[kSnapStages], kv_empty[kSnapStages];
    uint32_t tmem_base;
    alignas(16) float bias[256];  // per window column: m + log2(l) (log2 domain); +inf for invalid rows
    alignas(16) int pos[256];     // per window column: token position of its query row inside the group (-1: invalid)
    float2 stat[256];             // pass 1: (m, l) of the key-column half 1 of every window row, merged by half 0
    float part[2][3][128];        // pass-2 partial sums of column sets 1-3, by key tile parity
};
constexpr size_t kSnapSmem = 1024 + 2 * kSnapQChunk + kSnapStages * kSnapKTile + sizeof(SnapShared);

#ifdef QVK_SNAP_TRACE
// Developer timeline (tools/snap_trace.cu): clock64 per key tile of CTA 0's first two items.
//   [item][tile][0] MMA thread starts waiting acc_empty, [1] issues, [2] issued + committed
//   [3..5] warp 0 (set 0, quarter 0) lane 0: acc_full seen, accumulator released, tile's math done
//   [6..8] the same for warp 13 (set 3, quarter 1)
__device__ long long g_snap_trace[2][64][10];
__device__ unsigned long long g_snap_span[3];  // globaltimer: earliest CTA start, latest CTA end, CTA 0's first tile
#define QVK_ST(item_no, tile, slot)                                                       \
    do {                                                                                  \
        if (blockIdx.x == 0 && (item_no) < 2 && (tile) < 64) {                            \
            g_snap_trace[(item_no)][(tile)][(slot)] = clock64();                          \
            if ((slot) == 0) {                                                            \
                long long _g;                                                             \
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_g));                    \
                g_snap_trace[(item_no)][(tile)][9] = _g;                                  \
            }                                                                             \
        }                                                                                 \
    } while (0)
#else
#define QVK_ST(item_no, tile, slot) \
    do {                            \
    } while (0)
#endif

struct SnapParams {
    const int64_t* tok_off;
    int n_groups, n_kv, gq, window, rows, rows_pad;
    int wb, nb;  // window rows per block (rows = gq * wb <= 256) and blocks per item (nb * wb >= window)
    float sl2;
    const float* lse;  // optional: the window rows' softmax statistics from the attention kernel (skips pass 1)
    int after_attention;  // launched (PDL) while the attention that writes lse may still run: compute warps wait
    int tiles_flat;       // > 0 (pass 2 only, one window block): CTAs own equal ranges of the (item, key tile) space
                          // of tiles_flat tiles per item instead of whole items (pass-2 tiles are independent)
    float* raw;   // (group, head, token) layout, when pooling follows
    double* out;  // pool == 1: the double scores written directly (same value as the pool kernel's float -> double)
};

__device__ __forceinline__ uint64_t snap_desc(uint32_t chunk_addr, uint32_t chunk_stride, int kk) {
    // k-step kk (16 of the 128 head-dim columns) of a K-major SW128 operand stored as two d-chunks.
    return ptx::umma_desc_sw128(chunk_addr + (kk >> 2) * chunk_stride + (kk & 3) * 32, 16, 1024);
}

// The work segments of a CTA: whole (group, KV head) items round-robin, or — pass 2 alone, where every key tile is
// independent given the window statistics — a contiguous range of the items x tiles_flat key-tile space (C3: 2048
// tiles over 148 CTAs = 13-14 each instead of 1.73 waves of 8-tile items).  Every role walks the same segments.
struct SnapSegs {
    int64_t f1;
    int it, tm;
    int64_t f0;
    __device__ explicit SnapSegs(const SnapParams& p, int items) : tm(p.tiles_flat) {
        if (tm > 0) {
            const int64_t total = static_cast<int64_t>(items) * tm;
            f0 = total * blockIdx.x / gridDim.x;
            f1 = total * (blockIdx.x + 1) / gridDim.x;
            it = static_cast<int>(f0 / tm);
        } else {
            f0 = f1 = 0;
            it = blockIdx.x;
        }
    }
    // next segment: item, key tiles [jt0, jt1) (jt1 clipped to the group's tiles by the caller)
    __device__ bool next(int items, int& item, int& jt0, int& jt1) {
        if (tm > 0) {
            const int64_t base = static_cast<int64_t>(it) * tm;
            if (base >= f1 || it >= items) return false;
            item = it++;
            jt0 = static_cast<int>(f0 > base ? f0 - base : 0);
            jt1 = static_cast<int>(f1 - base < tm ? f1 - base : tm);
            return true;
        }
        if (it >= items) return false;
        item = it;
        it += gridDim.x;
        jt0 = 0;
        jt1 = 0x7fffffff;
        return true;
    }
};

// kN8: 8-column chunks of the pass-2 window columns per compute set (rows_pad = 32 kN8).
template <int kN8>
__global__ void __launch_bounds__(kSnapThreads, 1)
    snapkv_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                     const SnapParams p) {
    extern __shared__ uint8_t smem_raw[];
    // 1024-aligned window (SWIZZLE_128B atoms) by offsetting the shared array itself: the compiler keeps the shared
    // address space (LDS / STS, not generic LD / ST as through a uintptr_t round trip).
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sQ = smem;
    uint8_t* sK = smem + 2 * kSnapQChunk;
    SnapShared* sh = reinterpret_cast<SnapShared*>(sK + kSnapStages * kSnapKTile);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int items = p.n_groups * p.n_kv;
#ifdef QVK_SNAP_TRACE
    if (threadIdx.x == 0) {
        unsigned long long g0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
        atomicMin(&g_snap_span[0], g0);
    }
#endif

    if (threadIdx.x == 0) {
        ptx::mbar_init(&sh->q_full, 1);
        ptx::mbar_init(&sh->q_empty, 1);
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&sh->acc_full[b], 1);
            // pass 2 alone: a team of two compute sets (256 threads) per accumulator buffer
            ptx::mbar_init(&sh->acc_empty[b], p.lse ? kSnapCompute / 2 : kSnapCompute);
        }
        for (int st = 0; st < kSnapStages; ++st) {
            ptx::mbar_init(&sh->kv_full[st], 1);
            ptx::mbar_init(&sh->kv_empty[st], 1);
        }
        ptx::fence_mbar_init();
    }
    // Window-operand rows past gq * W are never written by the TMA (its box is exactly gq * W rows) but the
    // pass-2 MMA (N = rows_pad) and the pass-1 M-tile B read them: zero them once, so their columns of S' are 0 and
    // exp2(0 * scale - inf) = 0 exactly (stale smem could hold inf / nan bit patterns).
    if (p.rows < 256) {
        const int bytes = (256 - p.rows) * 128;
        for (int b = threadIdx.x * 16; b < bytes; b += kSnapThreads * 16) {
            *reinterpret_cast<uint4*>(sQ + p.rows * 128 + b) = make_uint4(0u, 0u, 0u, 0u);
            *reinterpret_cast<uint4*>(sQ + kSnapQChunk + p.rows * 128 + b) = make_uint4(0u, 0u, 0u, 0u);
        }
        ptx::fence_proxy_async_smem();  // generic-proxy stores -> read by the tensor core (async proxy)
    }
    if (warp == kSnapMmaWarp) ptx::tmem_alloc<512>(&sh->tmem_base);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = sh->tmem_base;

    if (warp == kSnapTmaWarp) {
        if (ptx::elect_one()) {  // ===== TMA producer =====
            uint32_t item_no = 0, tile_no = 0;
            SnapSegs segs(p, items);
            int it, jt0, jt1;
            while (segs.next(items, it, jt0, jt1))
              for (int b = 0; b < p.nb; ++b) {
                const int g = it / p.n_kv, hk = it - g * p.n_kv;
                const int64_t t0 = __ldg(p.tok_off + g);
                const int n = static_cast<int>(__ldg(p.tok_off + g + 1) - t0);
                const int nt = (n + 127) / 128;
                const int jte = min(jt1, nt);
                if (jt0 >= jte) continue;  // empty segment (every role skips it)
                ++item_no;
                ptx::mbar_wait(&sh->q_empty, ((item_no - 1) & 1) ^ 1);
                ptx::mbar_arrive_expect_tx(&sh->q_full, 2 * p.rows * 128);
                // window rows [b wb, b wb + wb): may start before the group or run past its end (rows masked)
                const int w0 = static_cast<int>(t0) + n - p.window + b * p.wb;
                ptx::tma_load_3d(sQ, &tm_q, &sh->q_full, 0, hk * p.gq, w0);
                ptx::tma_load_3d(sQ + kSnapQChunk, &tm_q, &sh->q_full, 64, hk * p.gq, w0);
                for (int pass = p.lse ? 1 : 0; pass < 2; ++pass)
                    for (int jt = pass ? jt0 : 0; jt < (pass ? jte : nt); ++jt, ++tile_no) {
                        const uint32_t st = tile_no % kSnapStages;
                        ptx::mbar_wait(&sh->kv_empty[st], ((tile_no / kSnapStages) & 1) ^ 1);
                        uint8_t* dst = sK + st * kSnapKTile;
                        ptx::mbar_arrive_expect_tx(&sh->kv_full[st], kSnapKTile);
                        const int row = static_cast<int>(t0) + jt * 128;
                        ptx::tma_load_3d(dst, &tm_k, &sh->kv_full[st], 0, hk, row);
                        ptx::tma_load_3d(dst + kSnapChunk, &tm_k, &sh->kv_full[st], 64, hk, row);
                    }
            }
        }
    } else if (warp == kSnapMmaWarp) {
        if (ptx::elect_one()) {  // ===== MMA issuer =====
            const uint32_t id1 = ptx::idesc_bf16_f32(128, 128, false, false);
            const uint32_t id2 = ptx::idesc_bf16_f32(128, p.rows_pad, false, false);
            const uint32_t q_addr = ptx::smem_u32(sQ), k_base = ptx::smem_u32(sK);
            uint32_t item_no = 0, tile_no = 0, acc_no = 0;
            SnapSegs segs(p, items);
            int it, jt0, jt1;
            while (segs.next(items, it, jt0, jt1))
              for (int b = 0; b < p.nb; ++b) {
                const int g = it / p.n_kv;
                const int n = static_cast<int>(__ldg(p.tok_off + g + 1) - __ldg(p.tok_off + g));
                const int nt = (n + 127) / 128;
                const int jte = min(jt1, nt);
                if (jt0 >= jte) continue;
                ptx::mbar_wait(&sh->q_full, item_no & 1);
                ++item_no;
                ptx::tc_fence_after();
                for (int pass = p.lse ? 1 : 0; pass < 2; ++pass)
                    for (int jt = pass ? jt0 : 0; jt < (pass ? jte : nt); ++jt, ++tile_no, ++acc_no) {
                        const uint32_t st = tile_no % kSnapStages;
#ifdef QVK_SNAP_TRACE
                        const int tr_tile = pass * nt + jt;
#endif
                        ptx::mbar_wait(&sh->kv_full[st], (tile_no / kSnapStages) & 1);
                        QVK_ST(item_no - 1, tr_tile, 0);
                        const uint32_t ab = acc_no & 1, acol = tmem + 256 * ab;  // accumulator buffer
                        ptx::mbar_wait(&sh->acc_empty[ab], ((acc_no >> 1) & 1) ^ 1);
                        QVK_ST(item_no - 1, tr_tile, 1);
                        ptx::tc_fence_after();
                        const uint32_t ka = k_base + st * kSnapKTile;
                        if (pass == 0) {
#pragma unroll
                            for (int kk = 0; kk < 8; ++kk) {
                                const uint64_t bk = snap_desc(ka, kSnapChunk, kk);
                                ptx::mma_ss(acol, snap_desc(q_addr, kSnapQChunk, kk), bk, id1, kk > 0);
                                ptx::mma_ss(acol + 128, snap_desc(q_addr + 128 * 128, kSnapQChunk, kk), bk, id1,
                                            kk > 0);
                            }
                        } else {
#pragma unroll
                            for (int kk = 0; kk < 8; ++kk)
                                ptx::mma_ss(acol, snap_desc(ka, kSnapChunk, kk),
                                            snap_desc(q_addr, kSnapQChunk, kk), id2, kk > 0);
                        }
                        ptx::mma_commit(&sh->kv_empty[st]);
                        ptx::mma_commit(&sh->acc_full[ab]);
                        if (pass == 1 && jt == jte - 1) ptx::mma_commit(&sh->q_empty);
                        QVK_ST(item_no - 1, tr_tile, 2);
                    }
            }
        }
    } else {
        // ===== compute: warps 0-15, set = warp / 4 (four warps, one per TMEM lane quarter) =====
        // Programmatic dependent launch behind the attention kernel: the TMA / MMA warps start on Q and K (inputs the
        // attention only reads) in its tail; the window statistics it writes are read only after this wait, which
        // also makes this grid's completion imply the attention's.
        if (p.after_attention) asm volatile("griddepcontrol.wait;" ::: "memory");
        const int set = warp >> 2, quarter = warp & 3;
        const int i = quarter * 32 + lane;  // TMEM lane
        const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
        const float sl2 = p.sl2;
        uint32_t acc_no = 0;
        // acc_full of accumulator acc_no + 1 is probed (non-blocking) halfway through the math of acc_no: the MMA has
        // usually finished by then, and the blocking try_wait at the next tile then costs a memory round trip (~300
        // cycles per tile, all four warps of a sub-partition at once; tools/snap_trace.cu) instead of nothing.
        bool ready = false;
        auto wait_acc = [&]() {
            if (!ready) ptx::mbar_wait(&sh->acc_full[acc_no & 1], (acc_no >> 1) & 1);
            ready = false;
        };
        auto probe_next = [&]() { ready = ptx::mbar_test(&sh->acc_full[(acc_no + 1) & 1], ((acc_no + 1) >> 1) & 1); };
#ifdef QVK_SNAP_TRACE
        const bool tr = (warp == 0 || warp == 13) && lane == 0;
        const int tr_o = warp == 0 ? 3 : 6;
        int tr_item = 0;
#define QVK_STC(tile, k) \
    do {                 \
        if (tr) QVK_ST(tr_item, (tile), tr_o + (k)); \
    } while (0)
#else
#define QVK_STC(tile, k) \
    do {                 \
    } while (0)
#endif
        const int mt = set & 1, ch = set >> 1;  // pass 1: M-tile (window rows 128 mt ..) and key-column half
        // pass 2: window columns [col0, col0 + 8 n8) — rows_pad split evenly over the four sets in 8-column chunks
        // (224 columns: 56 each; a 64 / 64 / 64 / 32 split left one set idle for a quarter of every tile)
        const int col0 = set * 8 * kN8;
        SnapSegs segs(p, items);
        int it, jt0, jt1;
        while (segs.next(items, it, jt0, jt1)) {
          const int g = it / p.n_kv, hk = it - g * p.n_kv;
          const int64_t t0 = __ldg(p.tok_off + g);
          const int n = static_cast<int>(__ldg(p.tok_off + g + 1) - t0);
          const int nt = (n + 127) / 128;
          const int jte = min(jt1, nt);
          if (jt0 >= jte) continue;
          for (int b = 0; b < p.nb; ++b) {
            // window column c = r * gq + h of block b -> window row b wb + r at token position n - W + b wb + r
            // (invalid when before the group or past the window)
            const int c_row = mt * 128 + i;
            const int wrow = b * p.wb + c_row / p.gq;
            const int my_pos = c_row < p.rows && wrow < p.window ? n - p.window + wrow : -1;
            if (p.lse) {  // pass 1 done by the attention kernel: its softmax statistics of the window rows
                if (ch == 0) {
                    sh->bias[c_row] = my_pos >= 0 ? -p.lse[(static_cast<int64_t>(g) * p.n_kv * p.gq + hk * p.gq +
                                                            c_row % p.gq) * p.window + wrow]
                                                  : -INFINITY;
                    sh->pos[c_row] = my_pos;
                }
                ptx::named_bar_sync(1, kSnapCompute);
            } else {
            // ---- pass 1: running max / sum of window row c_row over key columns [64 ch, 64 ch + 64) of each tile ----
            float m = -INFINITY, l = 0.f;
            for (int jt = 0; jt < nt; ++jt, ++acc_no) {
                wait_acc();
                QVK_STC(jt, 0);
                ptx::tc_fence_after();
                float x[64];
                const uint32_t col = tmem + lane_off + 256 * (acc_no & 1) + mt * 128 + ch * 64;
                QVK_TMEM_LD32F(col + 0, (x + 0));
                QVK_TMEM_LD32F(col + 32, (x + 32));
                ptx::tmem_ld_wait();
                ptx::tc_fence_before();
                ptx::mbar_arrive(&sh->acc_empty[acc_no & 1]);
                QVK_STC(jt, 1);
                if (my_pos >= 0) {
                    const int j0 = jt * 128 + ch * 64;
                    if (j0 > my_pos) continue;  // every key of this half lies after the row: all masked
                    if (j0 + 63 > my_pos) {
#pragma unroll
                        for (int c = 0; c < 64; ++c)
                            if (j0 + c > my_pos) x[c] = -INFINITY;
                    }
                    // four independent max / sum chains (the serial FMNMX / FADD chains were latency-bound)
                    float mx4[4] = {x[0], x[1], x[2], x[3]};
#pragma unroll
                    for (int c = 4; c < 64; ++c) mx4[c & 3] = fmaxf(mx4[c & 3], x[c]);
                    const float mx = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
                    const float mn = fmaxf(m, mx * sl2);
                    // packed pairs (FFMA2 / FADD2): the same fp32 operations per element, half the instructions
                    const ptx::f2 sl2x2 = ptx::f2_make(sl2, sl2), nmn2 = ptx::f2_make(-mn, -mn);
                    ptx::f2 sa = ptx::f2_make(0.f, 0.f), sb = sa;  // (s4[0], s4[1]), (s4[2], s4[3])
#pragma unroll
                    for (int c = 0; c < 64; c += 2) {
                        if (c == 32) probe_next();
                        float e0, e1;
                        ptx::f2_split(ptx::f2_fma(ptx::f2_make(x[c], x[c + 1]), sl2x2, nmn2), e0, e1);
                        if (kSnapPoly(c >> 1)) {
                            ptx::ex2_poly2(e0, e1);  // a share of the exponentials on the FMA pipe
                        } else {
                            e0 = ptx::ex2(e0);
                            e1 = ptx::ex2(e1);
                        }
                        if (c & 2) sb = ptx::f2_add(sb, ptx::f2_make(e0, e1));
                        else sa = ptx::f2_add(sa, ptx::f2_make(e0, e1));
                    }
                    float s0, s1, s2, s3;
                    ptx::f2_split(sa, s0, s1);
                    ptx::f2_split(sb, s2, s3);
                    const float sum = (s0 + s1) + (s2 + s3);
                    l = (m == -INFINITY ? 0.f : l * ptx::ex2(m - mn)) + sum;
                    m = mn;
                }
#ifdef QVK_SNAP_TRACE
                if (tr) asm volatile("" ::"f"(l));
#endif
                QVK_STC(jt, 2);
            }
            // merge the two key-column halves of every row: half 1 publishes (m, l), half 0 combines
            if (ch == 1) sh->stat[c_row] = make_float2(m, l);
            ptx::named_bar_sync(1, kSnapCompute);
            if (ch == 0) {
                const float2 o = sh->stat[c_row];
                const float mm = fmaxf(m, o.x);
                const float ll = (m == -INFINITY ? 0.f : l * ptx::ex2(m - mm)) + (o.x == -INFINITY ? 0.f : o.y * ptx::ex2(o.x - mm));
                sh->bias[c_row] = my_pos >= 0 ? -(mm + __log2f(ll)) : -INFINITY;  // negated: y = x scale + bias
                sh->pos[c_row] = my_pos;
            }
            ptx::named_bar_sync(1, kSnapCompute);
            }
            // ---- pass 2 alone (window statistics given): two teams of two compute sets take alternate key tiles —
            // team t the tiles of accumulator buffer t — so one team's TMEM loads and partial-sum exchange overlap
            // the other team's exponentials (with all four sets on every tile, the sub-partition's four warps ran
            // each tile's load / exponentials / exchange in lockstep: ~2200 cycles per tile for ~1344 of MUFU work).
            // A set covers two slices of 8 kN8 window columns, loaded one after the other into the same registers.
            if (p.lse) {
                const int team = set >> 1, sub = set & 1;
                const ptx::f2 sl2x2 = ptx::f2_make(sl2, sl2);
                for (int jt = jt0; jt < jte; ++jt, ++acc_no) {
                    if (static_cast<int>(acc_no & 1) != team) continue;
                    ptx::mbar_wait(&sh->acc_full[team], (acc_no >> 1) & 1);
                    ptx::tc_fence_after();
                    const int j = jt * 128 + i;
                    const bool edge = jt * 128 + 127 > n - p.window + b * p.wb;
                    ptx::f2 a01 = ptx::f2_make(0.f, 0.f), a23 = a01;
                    float x[8 * kN8];
#pragma unroll
                    for (int r = 0; r < 2; ++r) {
                        const int c0 = (2 * sub + r) * 8 * kN8;
#pragma unroll
                        for (int c8 = 0; c8 < kN8; ++c8)
                            QVK_TMEM_LD8F(tmem + lane_off + 256 * team + c0 + 8 * c8, (x + 8 * c8));
                        ptx::tmem_ld_wait();
                        if (r == 1) {  // both slices read: the MMA may refill this buffer
                            ptx::tc_fence_before();
                            ptx::mbar_arrive(&sh->acc_empty[team]);
                        }
                        const float4* b4 = reinterpret_cast<const float4*>(sh->bias + c0);
                        const int4* p4 = reinterpret_cast<const int4*>(sh->pos + c0);
                        auto col4 = [&](const float* xq, const float4 bb, const int4* pp, bool poly01, bool poly23) {
                            float y0, y1, y2, y3;
                            ptx::f2_split(ptx::f2_fma(ptx::f2_make(xq[0], xq[1]), sl2x2, ptx::f2_make(bb.x, bb.y)),
                                          y0, y1);
                            ptx::f2_split(ptx::f2_fma(ptx::f2_make(xq[2], xq[3]), sl2x2, ptx::f2_make(bb.z, bb.w)),
                                          y2, y3);
                            if (pp) {
                                const int4 pv = *pp;
                                if (j > pv.x) y0 = -INFINITY;
                                if (j > pv.y) y1 = -INFINITY;
                                if (j > pv.z) y2 = -INFINITY;
                                if (j > pv.w) y3 = -INFINITY;
                            }
                            if (poly01) {
                                ptx::ex2_poly2(y0, y1);
                            } else {
                                y0 = ptx::ex2(y0);
                                y1 = ptx::ex2(y1);
                            }
                            if (poly23) {
                                ptx::ex2_poly2(y2, y3);
                            } else {
                                y2 = ptx::ex2(y2);
                                y3 = ptx::ex2(y3);
                            }
                            a01 = ptx::f2_add(a01, ptx::f2_make(y0, y1));
                            a23 = ptx::f2_add(a23, ptx::f2_make(y2, y3));
                        };
                        if (edge) {
#pragma unroll
                            for (int e4 = 0; e4 < 2 * kN8; ++e4)
                                col4(x + 4 * e4, b4[e4], p4 + e4, kSnapPoly(2 * e4), kSnapPoly(2 * e4 + 1));
                        } else {
#pragma unroll
                            for (int e4 = 0; e4 < 2 * kN8; ++e4)
                                col4(x + 4 * e4, b4[e4], nullptr, kSnapPoly(2 * e4), kSnapPoly(2 * e4 + 1));
                        }
                    }
                    float a4[4];
                    ptx::f2_split(a01, a4[0], a4[1]);
                    ptx::f2_split(a23, a4[2], a4[3]);
                    const float acc = (a4[0] + a4[1]) + (a4[2] + a4[3]);
                    const uint32_t tp = (acc_no >> 1) & 1;  // the team's tile parity: part[] double-buffered
                    if (sub) sh->part[tp][team][i] = acc;
                    ptx::named_bar_sync(2 + 4 * team + quarter, 64);  // the two sets of this team and lane quarter
                    if (!sub && j < n) {
                        const float tot = acc + sh->part[tp][team][i];
                        const int64_t e = p.n_kv * t0 + static_cast<int64_t>(hk) * n + j;
                        const float t = b ? tot + (p.out ? static_cast<float>(p.out[e]) : p.raw[e]) : tot;
                        if (p.out) p.out[e] = static_cast<double>(t);
                        else p.raw[e] = t;
                    }
                }
            } else
            // ---- pass 2: key j = jt*128 + i, window columns [col0, col0 + 8 n8) ----
            for (int jt = jt0; jt < jte; ++jt, ++acc_no) {
                wait_acc();
                QVK_STC(nt + jt, 0);
                ptx::tc_fence_after();
                const int j = jt * 128 + i;
                const bool edge = jt * 128 + 127 > n - p.window + b * p.wb;  // some window rows precede some keys
                // load this set's 8-column chunks and release the accumulator BEFORE the exponentials, so the next key
                // tile's MMAs overlap them.  Columns past the window rows (up to rows_pad) have bias -inf: they add
                // exp2(-inf) = 0.
                float x[8 * kN8];
#pragma unroll
                for (int c8 = 0; c8 < kN8; ++c8)
                    QVK_TMEM_LD8F(tmem + lane_off + 256 * (acc_no & 1) + col0 + 8 * c8, (x + 8 * c8));
                ptx::tmem_ld_wait();
                ptx::tc_fence_before();
                ptx::mbar_arrive(&sh->acc_empty[acc_no & 1]);
                QVK_STC(nt + jt, 1);
                const ptx::f2 sl2x2 = ptx::f2_make(sl2, sl2);
                ptx::f2 a01 = ptx::f2_make(0.f, 0.f), a23 = a01;  // (a4[0], a4[1]), (a4[2], a4[3])
                // y = x * scale - (m + log2 l) of the column's window row, masked where the row precedes the key
                // (only on `edge` tiles: a warp-uniform branch keeps the compare off the other tiles)
                auto column4 = [&](const float* xq, const float4 bb, const int* pv, bool masked, bool poly01,
                                   bool poly23) {
                    float y0, y1, y2, y3;
                    ptx::f2_split(ptx::f2_fma(ptx::f2_make(xq[0], xq[1]), sl2x2, ptx::f2_make(bb.x, bb.y)), y0, y1);
                    ptx::f2_split(ptx::f2_fma(ptx::f2_make(xq[2], xq[3]), sl2x2, ptx::f2_make(bb.z, bb.w)), y2, y3);
                    if (masked) {
                        if (j > pv[0]) y0 = -INFINITY;
                        if (j > pv[1]) y1 = -INFINITY;
                        if (j > pv[2]) y2 = -INFINITY;
                        if (j > pv[3]) y3 = -INFINITY;
                    }
                    if (poly01) {  // a share of the exponentials on the FMA pipe
                        ptx::ex2_poly2(y0, y1);
                    } else {
                        y0 = ptx::ex2(y0);
                        y1 = ptx::ex2(y1);
                    }
                    if (poly23) {
                        ptx::ex2_poly2(y2, y3);
                    } else {
                        y2 = ptx::ex2(y2);
                        y3 = ptx::ex2(y3);
                    }
                    a01 = ptx::f2_add(a01, ptx::f2_make(y0, y1));
                    a23 = ptx::f2_add(a23, ptx::f2_make(y2, y3));
                };
                const float4* b4 = reinterpret_cast<const float4*>(sh->bias + col0);
                const int4* p4 = reinterpret_cast<const int4*>(sh->pos + col0);
                if (edge) {  // one warp-uniform branch around the whole unrolled loop keeps it one basic block
#pragma unroll
                    for (int e4 = 0; e4 < 2 * kN8; ++e4) {
                        if (e4 == kN8) probe_next();
                        const int4 pp = p4[e4];
                        const int pv[4] = {pp.x, pp.y, pp.z, pp.w};
                        column4(x + 4 * e4, b4[e4], pv, true, kSnapPoly(2 * e4), kSnapPoly(2 * e4 + 1));
                    }
                } else {
#pragma unroll
                    for (int e4 = 0; e4 < 2 * kN8; ++e4) {
                        if (e4 == kN8) probe_next();
                        column4(x + 4 * e4, b4[e4], nullptr, false, kSnapPoly(2 * e4), kSnapPoly(2 * e4 + 1));
                    }
                }
                float a4[4];
                ptx::f2_split(a01, a4[0], a4[1]);
                ptx::f2_split(a23, a4[2], a4[3]);
                const float acc = (a4[0] + a4[1]) + (a4[2] + a4[3]);
                QVK_STC(nt + jt, 2);
                if (set) sh->part[jt & 1][set - 1][i] = acc;
                ptx::named_bar_sync(2 + quarter, 128);  // the four sets of this lane quarter
                if (!set && j < n) {
                    const float tot = acc + ((sh->part[jt & 1][0][i] + sh->part[jt & 1][1][i]) + sh->part[jt & 1][2][i]);
                    const int64_t e = p.n_kv * t0 + static_cast<int64_t>(hk) * n + j;
                    // blocks after the first add to the earlier blocks' sum (same thread, program order; a
                    // double written from a float converts back exactly)
                    const float t = b ? tot + (p.out ? static_cast<float>(p.out[e]) : p.raw[e]) : tot;
                    if (p.out) p.out[e] = static_cast<double>(t);
                    else p.raw[e] = t;
                }
            }
            ptx::named_bar_sync(1, kSnapCompute);  // bias / pos / stat reused by the next item
#ifdef QVK_SNAP_TRACE
            ++tr_item;
#endif
          }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == kSnapMmaWarp) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tmem);
    }
#ifdef QVK_SNAP_TRACE
    if (threadIdx.x == 0) {
        unsigned long long g1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
        atomicMax(&g_snap_span[1], g1);
    }
#endif
}

bool snap_map(CUtensorMap* m, const void* base, int heads, int64_t tokens, uint32_t box_heads, uint32_t box_rows) {
    const auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(tensor_map_encoder());
    if (!enc) return false;
    cuuint64_t dims[3] = {128, static_cast<cuuint64_t>(heads), static_cast<cuuint64_t>(tokens)};
    cuuint64_t strides[2] = {256, static_cast<cuuint64_t>(heads) * 256};
    cuuint32_t box[3] = {64, box_heads, box_rows};
    cuuint32_t estr[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int kN8>
int launch_snap_tc(cudaStream_t stream, const CUtensorMap& mq, const CUtensorMap& mk, const SnapParams& sp,
                   unsigned grid) {
    QVK_CUDA_CHECK(func_attr(reinterpret_cast<const void*>(snapkv_tc_kernel<kN8>),
                             cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSnapSmem)));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kSnapThreads);
    cfg.dynamicSmemBytes = kSnapSmem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = sp.after_attention ? 1 : 0;
    QVK_CUDA_CHECK(cudaLaunchKernelEx(&cfg, snapkv_tc_kernel<kN8>, mq, mk, sp));
    return QVK_OK;
}

}  // namespace

int launch_snapkv(cudaStream_t stream, const qvk_groups* g, const void* q, const void* k, int n_q, int n_kv,
                  int d_h, int window, int pool, float scale, double* scores, const float* lse, int after_attention) {
    if (d_h != kD) {
        set_error("snapkv: only head_dim 128 is implemented");
        return QVK_E_UNSUPPORTED;
    }
    if (n_q <= 0 || n_kv <= 0 || n_q % n_kv) QVK_INVALID("snapkv: n_q must be a positive multiple of n_kv");
    if (window <= 0) QVK_INVALID("snapkv: window must be >= 1");
    if (pool < 1 || pool % 2 == 0) QVK_INVALID("snapkv: pool width must be odd and >= 1");
    if (g->total_tokens == 0) return QVK_OK;
    const float sl2 = scale * 1.4426950408889634f;
    float2* stats = nullptr;
    float* raw = nullptr;
    const int64_t total = g->total_tokens * n_kv;
    const int gq = n_q / n_kv;
    // tcgen05 path for every window: the gq * W window rows of a KV head are cut into nb blocks of gq * wb <= 256
    // operand rows (wb window rows each), run one after another by the CTA that owns the (group, KV head) item.
    const int per_block = std::max(1, 256 / gq);
    const int nb = (window + per_block - 1) / per_block;
    const int wb = (window + nb - 1) / nb;
    const bool tc = gq <= 256 && !env_knob("QVK_SNAPKV_SIMT", 0);
    const bool direct = tc && pool == 1;  // the tcgen05 kernel writes the double scores itself: no pool pass
    if (!direct) QVK_CUDA_CHECK(scratch_alloc(reinterpret_cast<void**>(&raw), sizeof(float) * total, stream));
    if (tc) {
        CUtensorMap mq, mk;
        if (!snap_map(&mq, q, n_q, g->total_tokens, static_cast<uint32_t>(gq), static_cast<uint32_t>(wb)) ||
            !snap_map(&mk, k, n_kv, g->total_tokens, 1, 128)) {
            if (raw) cudaFreeAsync(raw, stream);
            set_error("snapkv: cuTensorMapEncodeTiled failed");
            return QVK_E_CUDA;
        }

        SnapParams sp;
        sp.tok_off = g->tok_off_d;
        sp.n_groups = g->n_groups;
        sp.n_kv = n_kv;
        sp.gq = gq;
        sp.window = window;
        sp.wb = wb;
        sp.nb = nb;
        sp.rows = gq * wb;
        sp.rows_pad = (sp.rows + 31) / 32 * 32;
        sp.sl2 = sl2;
        sp.lse = lse;
        sp.after_attention = lse && after_attention && pool == 1;
        sp.raw = raw;
        sp.out = direct ? scores : nullptr;
        const int sms = sm_count();
        // pass 2 alone with one window block: split the (item, key tile) space evenly over the CTAs
        static const int flat_on = env_knob("QVK_SNAPKV_FLAT", 1);
        sp.tiles_flat = (lse && nb == 1 && flat_on) ? static_cast<int>((g->max_tokens + 127) / 128) : 0;
        const int64_t units = static_cast<int64_t>(g->n_groups) * n_kv * (sp.tiles_flat > 0 ? sp.tiles_flat : 1);
        const unsigned grid = static_cast<unsigned>(std::min<int64_t>(units, sms));
        int rc = QVK_OK;
        switch (sp.rows_pad / 32) {
            case 1: rc = launch_snap_tc<1>(stream, mq, mk, sp, grid); break;
            case 2: rc = launch_snap_tc<2>(stream, mq, mk, sp, grid); break;
            case 3: rc = launch_snap_tc<3>(stream, mq, mk, sp, grid); break;
            case 4: rc = launch_snap_tc<4>(stream, mq, mk, sp, grid); break;
            case 5: rc = launch_snap_tc<5>(stream, mq, mk, sp, grid); break;
            case 6: rc = launch_snap_tc<6>(stream, mq, mk, sp, grid); break;
            case 7: rc = launch_snap_tc<7>(stream, mq, mk, sp, grid); break;
            default: rc = launch_snap_tc<8>(stream, mq, mk, sp, grid); break;
        }
        if (rc != QVK_OK) {
            if (raw) cudaFreeAsync(raw, stream);
            return rc;
        }
        if (direct) return QVK_OK;
    } else {
    QVK_CUDA_CHECK(scratch_alloc(reinterpret_cast<void**>(&stats),
                                   sizeof(float2) * g->n_groups * n_q * static_cast<size_t>(window), stream));
    snap_stats_kernel<<<dim3(g->n_groups, n_q), 256, 0, stream>>>(
        static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(k), g->tok_off_d, n_q, n_kv, window,
        sl2, stats);
    QVK_LAUNCH_CHECK();
    const unsigned chunks = static_cast<unsigned>((g->max_tokens + 127) / 128);
    snap_colsum_kernel<<<dim3(g->n_groups, n_kv, chunks), 128, 0, stream>>>(
        static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(k), g->tok_off_d, n_q, n_kv, window,
        sl2, stats, raw);
    QVK_LAUNCH_CHECK();
    QVK_CUDA_CHECK(cudaFreeAsync(stats, stream));
    }
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, kNumSms * 16));
    snap_pool_kernel<<<blocks, 256, 0, stream>>>(raw, g->tok_off_d, g->n_groups, n_kv, total, pool, scores);
    QVK_LAUNCH_CHECK();
    QVK_CUDA_CHECK(cudaFreeAsync(raw, stream));
    return QVK_OK;
}

}  // namespace qvk
