// (a5)/(a6) importance-score kernels.  HBM-bound; exact (bit-identical to prefill.cpp:192-233).
//
// Norm scorers (prefill.cpp:200-212).  The reference sums double(x)^2 sequentially over the row; we reproduce that
// order exactly (one thread owns one (token, head) row and walks it j = 0..width-1 with __dmul_rn/__dadd_rn, which
// are never contracted into FMAs), so scores — and therefore the top-k index sets — are bit-identical, with no
// near-tie band.  The rows a CTA owns are contiguous in HBM, so the CTA stages them through shared memory with
// coalesced 16-byte loads in width chunks of 64 elements; each thread then reads its own padded smem row.
// Algorithmic bytes per (token, head): width*sizeof(T) read + 8 written.
#include <cudaTypedefs.h>

#include "common.cuh"
#include "ptx.cuh"

namespace qvk {
namespace {

constexpr int kScoreThreads = 128;  // rows (units) per CTA, one per thread
constexpr int kChunk = 64;          // elements of a row staged per step

template <typename T>
__device__ __forceinline__ double to_double(T x);
template <>
__device__ __forceinline__ double to_double<float>(float x) { return static_cast<double>(x); }
template <>
__device__ __forceinline__ double to_double<__nv_bfloat16>(__nv_bfloat16 x) {
    return static_cast<double>(__bfloat162float(x));
}

template <typename T>
__global__ void __launch_bounds__(kScoreThreads) score_norm_kernel(const T* __restrict__ x, int64_t units,
                                                                   int width, int heads,
                                                                   const int64_t* __restrict__ tok_off,
                                                                   int n_groups, int negate,
                                                                   double* __restrict__ out) {
    constexpr int kPad = sizeof(T) == 4 ? 1 : 2;  // odd 32-bit word stride -> conflict-free column reads
    constexpr int kStride = kChunk + kPad;
    constexpr int kVec = 16 / sizeof(T);          // elements per 16-byte load
    constexpr int kVecPerRow = kChunk / kVec;
    __shared__ T tile[kScoreThreads * kStride];

    const int64_t u0 = static_cast<int64_t>(blockIdx.x) * kScoreThreads;
    const int64_t left = units - u0;
    const int nu = left < kScoreThreads ? static_cast<int>(left) : kScoreThreads;
    const bool vec_ok = ((width * sizeof(T)) % 16 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
    const T* base = x + u0 * width;

    double sq = 0.0;
    for (int c0 = 0; c0 < width; c0 += kChunk) {
        const int cw = min(kChunk, width - c0);
        __syncthreads();
        if (vec_ok && cw == kChunk) {
            for (int v = threadIdx.x; v < nu * kVecPerRow; v += kScoreThreads) {
                const int r = v / kVecPerRow, q = v % kVecPerRow;
                const uint4 pkt = __ldg(reinterpret_cast<const uint4*>(base + static_cast<int64_t>(r) * width + c0) + q);
                const T* e = reinterpret_cast<const T*>(&pkt);
#pragma unroll
                for (int t = 0; t < kVec; ++t) tile[r * kStride + q * kVec + t] = e[t];
            }
        } else {
            for (int e = threadIdx.x; e < nu * cw; e += kScoreThreads) {
                const int r = e / cw, c = e - r * cw;
                tile[r * kStride + c] = base[static_cast<int64_t>(r) * width + c0 + c];
            }
        }
        __syncthreads();
        if (threadIdx.x < nu) {
            const T* row = tile + threadIdx.x * kStride;
            for (int c = 0; c < cw; ++c) {
                const double d = to_double(row[c]);
                sq = __dadd_rn(sq, __dmul_rn(d, d));  // prefill.cpp:207, never an FMA
            }
        }
    }
    if (threadIdx.x < nu) {
        const int64_t u = u0 + threadIdx.x;
        const int64_t t = u / heads;
        const int h = static_cast<int>(u - t * heads);
        const double norm = __dsqrt_rn(sq);
        const double s = negate ? -norm : norm;  // zero key -> -0.0 exactly like the reference
        if (heads == 1) {
            out[t] = s;
        } else {
            const int g = find_group(tok_off, n_groups, t);
            const int64_t t0 = __ldg(tok_off + g);
            const int64_t n = __ldg(tok_off + g + 1) - t0;
            out[heads * t0 + h * n + (t - t0)] = s;
        }
    }
}

// bf16 fast path: one thread per (token, head) row, the row read straight from HBM with kBatch 16-byte loads in
// flight per thread (a warp's loads cover 32 adjacent rows, so every fetched sector is used — the second half by
// the next load through L1), then summed in the reference's sequential order.  For bf16 inputs double(x)*double(x)
// is exact (16 significant bits), so fma(d, d, acc) rounds exactly like acc + d*d (prefill.cpp:207) — bit-identical.
constexpr int kSeqThreads = 256;

template <int kBatch>
__global__ void __launch_bounds__(kSeqThreads) score_norm_bf16_kernel(const __nv_bfloat16* __restrict__ x,
                                                                      int64_t units, int width, int heads,
                                                                      const int64_t* __restrict__ tok_off,
                                                                      int n_groups, int negate,
                                                                      double* __restrict__ out) {
    const int64_t u = static_cast<int64_t>(blockIdx.x) * kSeqThreads + threadIdx.x;
    if (u >= units) return;
    const uint4* row = reinterpret_cast<const uint4*>(x + u * width);
    const int chunks = width >> 3;
    double acc = 0.0;
    for (int c0 = 0; c0 < chunks; c0 += kBatch) {
        uint4 v[kBatch];
#pragma unroll
        for (int b = 0; b < kBatch; ++b) v[b] = c0 + b < chunks ? __ldg(row + c0 + b) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
        for (int b = 0; b < kBatch; ++b) {
            if (c0 + b >= chunks) break;
            const uint32_t w[4] = {v[b].x, v[b].y, v[b].z, v[b].w};
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const uint32_t bits = (q & 1) ? (w[q >> 1] & 0xffff0000u) : (w[q >> 1] << 16);
                const double d = static_cast<double>(__uint_as_float(bits));
                acc = __fma_rn(d, d, acc);
            }
        }
    }
    const double norm = __dsqrt_rn(acc);
    const double sc = negate ? -norm : norm;  // zero key -> -0.0 exactly like the reference
    if (heads == 1) {
        out[u] = sc;
    } else {
        const int64_t t = u / heads;
        const int hh = static_cast<int>(u - t * heads);
        const int g = find_group(tok_off, n_groups, t);
        const int64_t t0 = __ldg(tok_off + g);
        const int64_t n = __ldg(tok_off + g + 1) - t0;
        out[heads * t0 + hh * n + (t - t0)] = sc;
    }
}

// TMA-fed variant for per-head rows of 64 or 128 bf16 (every GQA configuration): 128-row tiles (16 or 32 KB,
// contiguous in HBM) stream into a 3-stage shared-memory ring through cp.async.bulk.tensor with the 128-byte
// swizzle, so each thread reads ITS row's 16-byte chunks bank-conflict-free (chunk c of row r sits at
// r*128 + ((c ^ (r & 7)) * 16)) while HBM sees fully coalesced bulk reads.  One producer warp, 4 consumer warps,
// 2 CTAs per SM, persistent over tiles; the per-row double sum is the reference's sequential order (exact, see
// score_norm_bf16_kernel).
constexpr int kTmaStages = 3;
constexpr int kTmaRows = 128;
constexpr int kTmaConsumers = 4 * kTmaRows;  // four threads per row

struct ScoreTmaShared {
    uint64_t full[kTmaStages], empty[kTmaStages];
};

// Reference-order (prefill.cpp:207) sum of squares of row r of a swizzled smem tile of NB 64-column boxes.
template <int NB>
__device__ double seq_sumsq_smem(uint32_t row_s, int r) {
    double acc = 0.0;
    for (int b = 0; b < NB; ++b)
        for (int c = 0; c < 8; ++c) {
            uint32_t w[4];
            ptx::lds128(w, row_s + b * kTmaRows * 128 + ((c ^ (r & 7)) << 4));
            for (int e = 0; e < 8; ++e) {
                const uint32_t bits = (e & 1) ? (w[e >> 1] & 0xffff0000u) : (w[e >> 1] << 16);
                const double d = static_cast<double>(__uint_as_float(bits));
                acc = __fma_rn(d, d, acc);
            }
        }
    return acc;
}

__device__ __forceinline__ void store_score(double* __restrict__ out, int64_t u, int heads, int g,
                                            const int64_t* __restrict__ tok_off, double sumsq, int negate) {
    const double norm = __dsqrt_rn(sumsq);
    const double sc = negate ? -norm : norm;  // zero row -> -0.0 exactly like the reference
    if (heads == 1) {
        out[u] = sc;
    } else {
        const int64_t tok = static_cast<uint32_t>(u) / heads;  // units < 2^31 on this path
        const int hh = static_cast<int>(u - tok * heads);
        const int64_t t0 = __ldg(tok_off + g);
        const int64_t n = __ldg(tok_off + g + 1) - t0;
        out[heads * t0 + hh * n + (tok - t0)] = sc;
    }
}

template <int NB>  // 64-element boxes per row (row width = 64 * NB)
__global__ void __launch_bounds__(kTmaConsumers + 32) score_norm_tma_kernel(
    const __grid_constant__ CUtensorMap tm, int64_t units, int heads, const int64_t* __restrict__ tok_off,
    int n_groups, int64_t max_tokens, int negate, double* __restrict__ out) {
    constexpr uint32_t kBox = kTmaRows * 128;        // bytes of one 64-column box
    constexpr uint32_t kTile = NB * kBox;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    ScoreTmaShared* sh = reinterpret_cast<ScoreTmaShared*>(smem + kTmaStages * kTile);
    const int warp = threadIdx.x >> 5;
    const int64_t tiles = (units + kTmaRows - 1) / kTmaRows;
    if (threadIdx.x == 0) {
        for (int st = 0; st < kTmaStages; ++st) {
            ptx::mbar_init(&sh->full[st], 1);
            ptx::mbar_init(&sh->empty[st], kTmaConsumers);
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();
    if (warp == kTmaConsumers / 32) {
        if (ptx::elect_one()) {
            ptx::prefetch_tmap(&tm);
            uint32_t k = 0;
            for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++k) {
                const uint32_t st = k % kTmaStages;
                ptx::mbar_wait(&sh->empty[st], ((k / kTmaStages) & 1) ^ 1);
                ptx::mbar_arrive_expect_tx(&sh->full[st], kTile);
#pragma unroll
                for (int b = 0; b < NB; ++b)
                    ptx::tma_load_2d(smem + st * kTile + b * kBox, &tm, &sh->full[st], 64 * b,
                                     static_cast<int>(t * kTmaRows));
            }
        }
        return;
    }
    // Four adjacent lanes share a row: lane quarter q reads the 16-byte chunks {2q, 2q+1} of every box (the
    // 8 lanes of a shared-memory phase then hit 8 distinct bank groups under the swizzle).
    const int r = threadIdx.x >> 2, q = threadIdx.x & 3;
    uint32_t k = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++k) {
        const uint32_t st = k % kTmaStages;
        ptx::mbar_wait(&sh->full[st], (k / kTmaStages) & 1);
        const uint8_t* row = smem + st * kTile + r * 128;
        // Partial sums in any order and, per row, the min / max 15-bit magnitude over the nonzero elements
        // (16x2 SIMD): if the row total S is below 2^(q_min + 53), q_min = 2 (E_min - 134) the exponent of a unit
        // dividing every bf16 square, every partial sum of ANY order is exact, so the result equals the
        // reference's sequential sum bit for bit.  Rows that fail the test (huge dynamic range, inf / nan) are
        // recomputed sequentially.
        double acc[2] = {0.0, 0.0};
        uint32_t lo = 0xffffffffu;  // min(|x| - 1) over the row (zero wraps to the max: ignored), fp32 bits
        const uint32_t row_s = ptx::smem_u32(row);
#pragma unroll
        for (int b = 0; b < NB; ++b)
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
                const int c = 2 * q + cc;
                uint32_t w[4];
                ptx::lds128(w, row_s + b * kBox + ((c ^ (r & 7)) << 4));
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const uint32_t bits = (e & 1) ? (w[e >> 1] & 0xffff0000u) : (w[e >> 1] << 16);
                    lo = min(lo, (bits & 0x7fffffffu) - 1u);
                    const double d = static_cast<double>(__uint_as_float(bits));
                    acc[e & 1] = __fma_rn(d, d, acc[e & 1]);
                }
            }
        double sum = __dadd_rn(acc[0], acc[1]);
#pragma unroll
        for (int o = 1; o < 4; o <<= 1) {
            sum = __dadd_rn(sum, __shfl_xor_sync(0xffffffffu, sum, o));
            lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        }
        // Exactness test: every bf16 square is a multiple of 2^q, q = 2 (E - 134) with E the bf16 exponent
        // (E >= 1; (|x|-1) >> 23 underestimates it by at most one, which only makes the test conservative).
        // inf / nan elements make the sum non-finite: recomputed sequentially too (payload and sign included).
        const uint64_t sum_bits = static_cast<uint64_t>(__double_as_longlong(sum));
        bool exact = ((sum_bits >> 52) & 0x7ff) != 0x7ff;
        if (exact && lo != 0xffffffffu) {
            const int qmin = 2 * (static_cast<int>(lo >> 23) - 134);
            const int es = static_cast<int>((__double_as_longlong(sum) >> 52) & 0x7ff) - 1023;
            exact = es <= qmin + 52;
        }
        if (!exact && q == 0) sum = seq_sumsq_smem<NB>(row_s, r);  // rare: prefill.cpp:207's sequential order
        ptx::mbar_arrive(&sh->empty[st]);
        const int64_t u = t * kTmaRows + r;
        if (q == 0 && u < units)
            store_score(out, u, heads,
                        heads == 1 ? 0 : find_group_fast(tok_off, n_groups, static_cast<uint32_t>(u) / heads, max_tokens),
                        tok_off, sum, negate);
    }
}

bool score_map(CUtensorMap* m, const void* base, int64_t units, int width) {
    const auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(tensor_map_encoder());
    if (!enc) return false;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(width), static_cast<cuuint64_t>(units)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(width) * 2};
    cuuint32_t box[2] = {64, static_cast<cuuint32_t>(kTmaRows)};
    cuuint32_t estr[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int NB>
int launch_score_tma(cudaStream_t stream, const CUtensorMap& tm, int64_t units, int heads, const qvk_groups* g,
                     int negate, double* scores) {
    constexpr size_t smem = 1024 + kTmaStages * NB * kTmaRows * 128 + sizeof(ScoreTmaShared);
    QVK_CUDA_CHECK(func_attr(reinterpret_cast<const void*>(score_norm_tma_kernel<NB>),
                             cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    const int sms = sm_count();
    const int64_t tiles = (units + kTmaRows - 1) / kTmaRows;
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(tiles, 2 * static_cast<int64_t>(sms)));
    score_norm_tma_kernel<NB><<<grid, kTmaConsumers + 32, smem, stream>>>(tm, units, heads, g->tok_off_d,
                                                                          g->n_groups, g->max_tokens, negate, scores);
    QVK_LAUNCH_CHECK();
    return QVK_OK;
}

// attention_score (prefill.cpp:213-230): s_i = (sum_t sum_j double(k_ij) * q_tj) / (T * n_h), t-outer, j-inner,
// one running double — reproduced in the same order.  q rows are read by every thread at the same time (broadcast);
// each thread walks its own key row (L1-resident across the t loop).
template <typename T>
__global__ void __launch_bounds__(128) score_attention_kernel(const T* __restrict__ k, int64_t tokens, int d,
                                                              const float* __restrict__ q, int64_t text_count,
                                                              double divisor, double* __restrict__ out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= tokens) return;
    const T* key = k + i * d;
    double sum = 0.0;
    for (int64_t t = 0; t < text_count; ++t) {
        const float* qt = q + t * d;
        for (int j = 0; j < d; ++j)
            sum = __dadd_rn(sum, __dmul_rn(to_double(key[j]), static_cast<double>(__ldg(qt + j))));
    }
    out[i] = __ddiv_rn(sum, divisor);
}

// Same sum, with each thread's key row staged in shared memory (row stride d + 1 words: conflict-free column reads)
// and the text-query element broadcast: the sequential t-outer / j-inner double chain of prefill.cpp:220-226 is then
// bound by the DADD latency instead of an L1/L2 miss per element (the per-thread rows of the kernel above do not fit
// L1).  R rows (threads) per CTA, R = min(32, what fits in 96 KB).
template <typename T>
__global__ void score_attention_smem_kernel(const T* __restrict__ k, int64_t tokens, int d,
                                            const float* __restrict__ q, int64_t text_count, double divisor,
                                            double* __restrict__ out) {
    extern __shared__ float srow[];  // [R][d + 1]
    const int R = blockDim.x;
    const int64_t i0 = static_cast<int64_t>(blockIdx.x) * R;
    const int nr = static_cast<int>(tokens - i0 < R ? tokens - i0 : R);
    for (int e = threadIdx.x; e < nr * d; e += R) {
        const int r = e / d, c = e - r * d;
        srow[r * (d + 1) + c] = static_cast<float>(k[(i0 + r) * d + c]);
    }
    __syncthreads();
    if (threadIdx.x >= nr) return;
    const float* key = srow + threadIdx.x * (d + 1);
    double sum = 0.0;
    for (int64_t t = 0; t < text_count; ++t) {
        const float* qt = q + t * d;
#pragma unroll 8
        for (int j = 0; j < d; ++j)
            sum = __dadd_rn(sum, __dmul_rn(static_cast<double>(key[j]), static_cast<double>(__ldg(qt + j))));
    }
    out[i0 + threadIdx.x] = __ddiv_rn(sum, divisor);
}

// ---- GQA attention_score on a pre-summed text query (qvk_score_text, include/qvk.h) ------------------------------
// qbar[h, j] = float(sum_t sum_{hq in group(h)} double(q[t, hq, j])), t outer, hq inner — one thread per (h, j).
__global__ void text_query_sum_kernel(const float* __restrict__ q, int64_t text_count, int n_q, int n_kv, int d_h,
                                      float* __restrict__ qbar) {
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= n_kv * d_h) return;
    const int h = o / d_h, j = o - h * d_h, gq = n_q / n_kv;
    double acc = 0.0;
    for (int64_t t = 0; t < text_count; ++t)
        for (int x = 0; x < gq; ++x)
            acc = __dadd_rn(acc, static_cast<double>(__ldg(q + (t * n_q + h * gq + x) * d_h + j)));
    qbar[o] = static_cast<float>(acc);
}

// s = (sum_j double(k_j) * double(qbar_j)) / divisor over one (token, head) row, j sequential (prefill.cpp:220-226
// with a single text row).  bf16 x fp32 products are exact in double, so fma(k, q, acc) rounds exactly like
// acc + k*q: bit-identical to the reference's loop on the same row.  Generic widths: the row is read straight from
// HBM (16-byte loads when aligned).
__device__ __forceinline__ void store_unit(double* __restrict__ out, int64_t u, int heads, int n_groups,
                                           const int64_t* __restrict__ tok_off, int64_t stride, double s) {
    if (heads == 1) {
        out[u] = s;
        return;
    }
    const int64_t tok = u / heads;
    const int hh = static_cast<int>(u - tok * heads);
    const int g = find_group_fast(tok_off, n_groups, tok, stride);
    const int64_t t0 = __ldg(tok_off + g);
    const int64_t n = __ldg(tok_off + g + 1) - t0;
    out[heads * t0 + hh * n + (tok - t0)] = s;
}

__global__ void __launch_bounds__(kSeqThreads) score_dot_seq_kernel(const __nv_bfloat16* __restrict__ k,
                                                                    int64_t units, int width, int heads,
                                                                    const float* __restrict__ qbar, double divisor,
                                                                    const int64_t* __restrict__ tok_off, int n_groups,
                                                                    int64_t max_tokens, double* __restrict__ out) {
    const int64_t u = static_cast<int64_t>(blockIdx.x) * kSeqThreads + threadIdx.x;
    if (u >= units) return;
    const int h = static_cast<int>(u % heads);
    const __nv_bfloat16* row = k + u * width;
    const float* qb = qbar + static_cast<int64_t>(h) * width;
    double acc = 0.0;
    if ((width & 7) == 0 && (reinterpret_cast<uintptr_t>(k) & 15) == 0) {
        for (int c = 0; c < width / 8; ++c) {
            const uint4 p = __ldg(reinterpret_cast<const uint4*>(row) + c);
            const uint32_t w[4] = {p.x, p.y, p.z, p.w};
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const uint32_t bits = (e & 1) ? (w[e >> 1] & 0xffff0000u) : (w[e >> 1] << 16);
                acc = __fma_rn(static_cast<double>(__uint_as_float(bits)),
                               static_cast<double>(__ldg(qb + c * 8 + e)), acc);
            }
        }
    } else {
        for (int j = 0; j < width; ++j)
            acc = __fma_rn(to_double(row[j]), static_cast<double>(__ldg(qb + j)), acc);
    }
    store_unit(out, u, heads, n_groups, tok_off, max_tokens, __ddiv_rn(acc, divisor));
}

// Per-head rows of 64 / 128 bf16 (every GQA shape): the norm kernel's TMA ring (128-row tiles, 128-byte swizzle,
// one producer warp) with ONE consumer thread per row walking its row j = 0..W-1 (chunk c of row r sits at
// r*128 + ((c ^ (r & 7)) * 16): conflict-free), qbar held as doubles in shared memory with a padded per-head stride
// (the heads of one warp's rows read distinct banks).  HBM-bound: N*W*2 bytes read, N*8 written.
constexpr int kDotConsumers = kTmaRows;

template <int NB>
__global__ void __launch_bounds__(kDotConsumers + 32) score_dot_tma_kernel(
    const __grid_constant__ CUtensorMap tm, int64_t units, int heads, const float* __restrict__ qbar,
    double divisor, const int64_t* __restrict__ tok_off, int n_groups, int64_t max_tokens, double* __restrict__ out) {
    constexpr int W = 64 * NB;
    constexpr int kQStride = W + 1;                  // doubles per head row of qbar in smem
    constexpr uint32_t kBox = kTmaRows * 128;
    constexpr uint32_t kTile = NB * kBox;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    ScoreTmaShared* sh = reinterpret_cast<ScoreTmaShared*>(smem + kTmaStages * kTile);
    double* qs = reinterpret_cast<double*>(sh + 1);  // [heads][kQStride]
    const int warp = threadIdx.x >> 5;
    const int64_t tiles = (units + kTmaRows - 1) / kTmaRows;
    for (int i = threadIdx.x; i < heads * W; i += blockDim.x)
        qs[(i / W) * kQStride + (i % W)] = static_cast<double>(__ldg(qbar + i));
    if (threadIdx.x == 0) {
        for (int st = 0; st < kTmaStages; ++st) {
            ptx::mbar_init(&sh->full[st], 1);
            ptx::mbar_init(&sh->empty[st], kDotConsumers);
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();
    if (warp == kDotConsumers / 32) {
        if (ptx::elect_one()) {
            ptx::prefetch_tmap(&tm);
            uint32_t k = 0;
            for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++k) {
                const uint32_t st = k % kTmaStages;
                ptx::mbar_wait(&sh->empty[st], ((k / kTmaStages) & 1) ^ 1);
                ptx::mbar_arrive_expect_tx(&sh->full[st], kTile);
#pragma unroll
                for (int b = 0; b < NB; ++b)
                    ptx::tma_load_2d(smem + st * kTile + b * kBox, &tm, &sh->full[st], 64 * b,
                                     static_cast<int>(t * kTmaRows));
            }
        }
        return;
    }
    const int r = threadIdx.x;
    uint32_t k = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++k) {
        const uint32_t st = k % kTmaStages;
        ptx::mbar_wait(&sh->full[st], (k / kTmaStages) & 1);
        const int64_t u = t * kTmaRows + r;
        const double* q = qs + static_cast<int>(u % heads) * kQStride;
        const uint32_t row_s = ptx::smem_u32(smem + st * kTile + r * 128);
        double acc = 0.0;
#pragma unroll
        for (int b = 0; b < NB; ++b)
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                uint32_t w[4];
                ptx::lds128(w, row_s + b * kBox + ((c ^ (r & 7)) << 4));
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const uint32_t bits = (e & 1) ? (w[e >> 1] & 0xffff0000u) : (w[e >> 1] << 16);
                    acc = __fma_rn(static_cast<double>(__uint_as_float(bits)), q[b * 64 + c * 8 + e], acc);
                }
            }
        ptx::mbar_arrive(&sh->empty[st]);
        if (u < units) store_unit(out, u, heads, n_groups, tok_off, max_tokens, __ddiv_rn(acc, divisor));
    }
}

}  // namespace

int launch_score(cudaStream_t stream, const qvk_groups* g, int64_t total_tokens, const void* k, const void* v,
                 int dtype, int heads, int width, int scorer, const float* text_query, int64_t text_count,
                 int n_h, double* scores) {
    if (scorer == QVK_KEY_NORM_SMALL || scorer == QVK_VALUE_NORM) {
        const void* x = scorer == QVK_KEY_NORM_SMALL ? k : v;
        const int64_t units = total_tokens * heads;
        if (units == 0) return QVK_OK;
        const unsigned blocks = static_cast<unsigned>((units + kScoreThreads - 1) / kScoreThreads);
        const int negate = scorer == QVK_KEY_NORM_SMALL;
        const bool fast = dtype == QVK_BF16 && width % 8 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0;
        CUtensorMap tm;
        if (fast && (width == 64 || width == 128) && units < (int64_t(1) << 31) && score_map(&tm, x, units, width)) {
            return width == 64 ? launch_score_tma<1>(stream, tm, units, heads, g, negate, scores)
                               : launch_score_tma<2>(stream, tm, units, heads, g, negate, scores);
        }
        if (fast) {
            const unsigned grid = static_cast<unsigned>((units + kSeqThreads - 1) / kSeqThreads);
            const auto* xb = static_cast<const __nv_bfloat16*>(x);
            if (width <= 64)
                score_norm_bf16_kernel<8><<<grid, kSeqThreads, 0, stream>>>(xb, units, width, heads, g->tok_off_d,
                                                                            g->n_groups, negate, scores);
            else
                score_norm_bf16_kernel<16><<<grid, kSeqThreads, 0, stream>>>(xb, units, width, heads, g->tok_off_d,
                                                                             g->n_groups, negate, scores);
        } else if (dtype == QVK_F32)
            score_norm_kernel<float><<<blocks, kScoreThreads, 0, stream>>>(
                static_cast<const float*>(x), units, width, heads, g->tok_off_d, g->n_groups, negate, scores);
        else
            score_norm_kernel<__nv_bfloat16><<<blocks, kScoreThreads, 0, stream>>>(
                static_cast<const __nv_bfloat16*>(x), units, width, heads, g->tok_off_d, g->n_groups, negate,
                scores);
        QVK_LAUNCH_CHECK();
        return QVK_OK;
    }
    if (scorer == QVK_ATTENTION_SCORE) {
        if (heads != 1) QVK_INVALID("attention_score: per-token mode only (heads must be 1)");
        if (total_tokens == 0) return QVK_OK;
        const unsigned blocks = static_cast<unsigned>((total_tokens + 127) / 128);
        const double divisor = static_cast<double>(text_count) * static_cast<double>(n_h);
        const int rows = std::min<int>(32, static_cast<int>((96 * 1024) / ((static_cast<size_t>(width) + 1) * 4)));
        if (rows >= 1) {  // staged-row kernel (every width up to 24575)
            const size_t smem = static_cast<size_t>(rows) * (width + 1) * sizeof(float);
            const unsigned grid = static_cast<unsigned>((total_tokens + rows - 1) / rows);
            if (dtype == QVK_F32) {
                QVK_CUDA_CHECK(func_attr(reinterpret_cast<const void*>(score_attention_smem_kernel<float>),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
                score_attention_smem_kernel<float><<<grid, rows, smem, stream>>>(
                    static_cast<const float*>(k), total_tokens, width, text_query, text_count, divisor, scores);
            } else {
                QVK_CUDA_CHECK(func_attr(reinterpret_cast<const void*>(score_attention_smem_kernel<__nv_bfloat16>),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
                score_attention_smem_kernel<__nv_bfloat16><<<grid, rows, smem, stream>>>(
                    static_cast<const __nv_bfloat16*>(k), total_tokens, width, text_query, text_count, divisor,
                    scores);
            }
            QVK_LAUNCH_CHECK();
            return QVK_OK;
        }
        if (dtype == QVK_F32)
            score_attention_kernel<float><<<blocks, 128, 0, stream>>>(static_cast<const float*>(k), total_tokens,
                                                                     width, text_query, text_count, divisor, scores);
        else
            score_attention_kernel<__nv_bfloat16><<<blocks, 128, 0, stream>>>(
                static_cast<const __nv_bfloat16*>(k), total_tokens, width, text_query, text_count, divisor, scores);
        QVK_LAUNCH_CHECK();
        return QVK_OK;
    }
    QVK_INVALID("score: unknown scorer");
}

int launch_text_query_sum(cudaStream_t stream, const float* q, int64_t text_count, int n_q, int n_kv, int d_h,
                          float* qbar) {
    const int n = n_kv * d_h;
    text_query_sum_kernel<<<(n + 127) / 128, 128, 0, stream>>>(q, text_count, n_q, n_kv, d_h, qbar);
    QVK_LAUNCH_CHECK();
    return QVK_OK;
}

// Scores of every (token, head) row of k (heads x width bf16) against qbar (heads x width fp32), divided by divisor.
int launch_score_dot(cudaStream_t stream, const qvk_groups* g, const void* k, int heads, int width,
                     const float* qbar, double divisor, double* scores) {
    const int64_t units = g->total_tokens * heads;
    if (units == 0) return QVK_OK;
    CUtensorMap tm;
    if ((width == 64 || width == 128) && heads <= 16 && (reinterpret_cast<uintptr_t>(k) & 15) == 0 &&
        units < (int64_t(1) << 31) && score_map(&tm, k, units, width)) {
        auto go = [&](auto kern, int nb) -> int {
            const size_t smem = 1024 + kTmaStages * nb * kTmaRows * 128 + sizeof(ScoreTmaShared) +
                                static_cast<size_t>(heads) * (64 * nb + 1) * sizeof(double);
            QVK_CUDA_CHECK(func_attr(reinterpret_cast<const void*>(kern), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
            const int64_t tiles = (units + kTmaRows - 1) / kTmaRows;
            const unsigned grid = static_cast<unsigned>(std::min<int64_t>(tiles, 2 * static_cast<int64_t>(sm_count())));
            kern<<<grid, kDotConsumers + 32, smem, stream>>>(tm, units, heads, qbar, divisor, g->tok_off_d,
                                                            g->n_groups, g->max_tokens, scores);
            QVK_LAUNCH_CHECK();
            return QVK_OK;
        };
        return width == 64 ? go(score_dot_tma_kernel<1>, 1) : go(score_dot_tma_kernel<2>, 2);
    }
    const unsigned grid = static_cast<unsigned>((units + kSeqThreads - 1) / kSeqThreads);
    score_dot_seq_kernel<<<grid, kSeqThreads, 0, stream>>>(static_cast<const __nv_bfloat16*>(k), units, width, heads,
                                                           qbar, divisor, g->tok_off_d, g->n_groups, g->max_tokens,
                                                           scores);
    QVK_LAUNCH_CHECK();
    return QVK_OK;
}

}  // namespace qvk
