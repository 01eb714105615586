// (a7) SnapKV observation-window scores (north star (3); no reference code — DESIGN.md §3.3 states the definition):
//   window rows r in [N - W, N), W = min(window, N); for KV head h and each of its n_q/n_kv query heads:
//   s[h, j] += causal softmax_j(scale * q_r . k_j)  (j <= r);  optional average pooling (odd width, zero padded).
// Two passes over K per (group, head): (1) per window row max/sum of the causal logits, (2) per key the sum of the
// normalised probabilities.  fp32 FMA on CUDA cores; HBM reads of K are the algorithmic bytes
// (N * d * 2 + W * n_q * d * 2 read, N * n_kv * 8 written per group).
#include "common.cuh"

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

}  // namespace

int launch_snapkv(cudaStream_t stream, const qvk_groups* g, const void* q, const void* k, int n_q, int n_kv,
                  int d_h, int window, int pool, float scale, double* scores) {
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
    QVK_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&stats),
                                   sizeof(float2) * g->n_groups * n_q * static_cast<size_t>(window), stream));
    QVK_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&raw), sizeof(float) * total, stream));
    snap_stats_kernel<<<dim3(g->n_groups, n_q), 256, 0, stream>>>(
        static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(k), g->tok_off_d, n_q, n_kv, window,
        sl2, stats);
    QVK_LAUNCH_CHECK();
    const unsigned chunks = static_cast<unsigned>((g->max_tokens + 127) / 128);
    snap_colsum_kernel<<<dim3(g->n_groups, n_kv, chunks), 128, 0, stream>>>(
        static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(k), g->tok_off_d, n_q, n_kv, window,
        sl2, stats, raw);
    QVK_LAUNCH_CHECK();
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, kNumSms * 16));
    snap_pool_kernel<<<blocks, 256, 0, stream>>>(raw, g->tok_off_d, g->n_groups, n_kv, total, pool, scores);
    QVK_LAUNCH_CHECK();
    QVK_CUDA_CHECK(cudaFreeAsync(stats, stream));
    QVK_CUDA_CHECK(cudaFreeAsync(raw, stream));
    return QVK_OK;
}

}  // namespace qvk
