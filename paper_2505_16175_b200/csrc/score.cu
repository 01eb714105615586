// (a5)/(a6) importance-score kernels.  HBM-bound; exact (bit-identical to prefill.cpp:192-233).
//
// Norm scorers (prefill.cpp:200-212).  The reference sums double(x)^2 sequentially over the row; we reproduce that
// order exactly (one thread owns one (token, head) row and walks it j = 0..width-1 with __dmul_rn/__dadd_rn, which
// are never contracted into FMAs), so scores — and therefore the top-k index sets — are bit-identical, with no
// near-tie band.  The rows a CTA owns are contiguous in HBM, so the CTA stages them through shared memory with
// coalesced 16-byte loads in width chunks of 64 elements; each thread then reads its own padded smem row.
// Algorithmic bytes per (token, head): width*sizeof(T) read + 8 written.
#include "common.cuh"

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

}  // namespace qvk
