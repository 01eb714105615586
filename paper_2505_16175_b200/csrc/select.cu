// (a9) top-k selection: one CTA per (group, head) segment, exact radix select on 64-bit order-preserving keys.
//
// Semantics (prefill.cpp:240-253): the k best scores under the strict order (score desc, index asc), -0.0 == +0.0,
// returned as ascending indices.  Algorithm:
//   1. keys = score_key(score) (common.cuh), cached in shared memory when the segment fits (else re-read);
//   2. MSB-first radix select, 8 bits per pass: a warp-aggregated shared histogram of the next digit among keys
//      that match the resolved prefix, a 256-bin suffix scan to pick the digit holding the k-th key; stop early once
//      the chosen bucket is taken whole;
//   3. ascending compaction: a key is kept iff its resolved prefix is above the threshold, or equal to it and it is
//      among the first `need` equal keys by index — two block-wide scans (equal-rank, then output slot).
// The result is identical to std::nth_element + std::sort under the reference's comparator.
#include "common.cuh"

namespace qvk {
namespace {

constexpr int kSelThreads = 512;
constexpr int kSelWarps = kSelThreads / 32;

struct SelShared {
    uint32_t hist[256];
    uint32_t warp[kSelWarps];
    uint64_t prefix;
    uint32_t need;
    uint32_t bucket;
};

// Exclusive block scan of v; *total gets the block sum.  All threads must call.
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* warp_sums, uint32_t* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t n = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += n;
    }
    if (lane == 31) warp_sums[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        uint32_t w = lane < kSelWarps ? warp_sums[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t n = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += n;
        }
        if (lane < kSelWarps) warp_sums[lane] = w;  // inclusive warp totals
    }
    __syncthreads();
    const uint32_t before = wid ? warp_sums[wid - 1] : 0u;
    *total = warp_sums[kSelWarps - 1];
    __syncthreads();  // warp_sums reusable after return
    return before + incl - v;
}

template <bool kSmem>
__global__ void __launch_bounds__(kSelThreads) select_kernel(const double* __restrict__ scores,
                                                             const int64_t* __restrict__ tok_off,
                                                             const int64_t* __restrict__ keep,
                                                             const int64_t* __restrict__ row_off, int heads,
                                                             uint32_t* __restrict__ idx_out) {
    extern __shared__ __align__(16) uint64_t skeys[];
    __shared__ SelShared sh;

    const int g = blockIdx.x / heads;
    const int h = blockIdx.x - g * heads;
    const int64_t t0 = tok_off[g];
    const int n = static_cast<int>(tok_off[g + 1] - t0);
    const double* s = scores + heads * t0 + static_cast<int64_t>(h) * n;
    const int64_t kk = keep[g];
    const int k = kk < n ? static_cast<int>(kk) : n;
    uint32_t* out = idx_out + row_off[g] * heads + h;
    if (k <= 0) return;
    if (k == n) {  // everything kept, in order
        for (int i = threadIdx.x; i < n; i += kSelThreads) out[static_cast<int64_t>(i) * heads] = i;
        return;
    }
    if (kSmem)
        for (int i = threadIdx.x; i < n; i += kSelThreads) skeys[i] = score_key(__ldg(s + i));
    auto key_at = [&](int i) -> uint64_t { return kSmem ? skeys[i] : score_key(__ldg(s + i)); };

    const int lane = threadIdx.x & 31;
    uint64_t prefix = 0, mask = 0;
    uint32_t need = static_cast<uint32_t>(k);
    const int rounds = (n + kSelThreads - 1) / kSelThreads;
    for (int shift = 56; shift >= 0; shift -= 8) {
        if (threadIdx.x < 256) sh.hist[threadIdx.x] = 0;
        __syncthreads();
        for (int rd = 0; rd < rounds; ++rd) {
            const int i = rd * kSelThreads + threadIdx.x;
            uint32_t digit = 0xffffffffu;  // sentinel: not a candidate
            if (i < n) {
                const uint64_t key = key_at(i);
                if ((key & mask) == prefix) digit = static_cast<uint32_t>(key >> shift) & 255u;
            }
            const uint32_t peers = __match_any_sync(0xffffffffu, digit);
            if (digit != 0xffffffffu && lane == __ffs(peers) - 1) atomicAdd(&sh.hist[digit], __popc(peers));
        }
        __syncthreads();
        // Suffix scan over bins: thread t (< 256) looks at bin b = 255 - t; incl = #candidates in bins >= b.
        uint32_t c = 0;
        if (threadIdx.x < 256) c = sh.hist[255 - threadIdx.x];
        uint32_t total;
        const uint32_t excl = block_exclusive_scan(c, sh.warp, &total);
        if (threadIdx.x < 256 && excl < need && excl + c >= need) {
            sh.prefix = prefix | (static_cast<uint64_t>(255 - threadIdx.x) << shift);
            sh.need = need - excl;
            sh.bucket = c;
        }
        __syncthreads();
        prefix = sh.prefix;
        need = sh.need;
        mask |= 0xffull << shift;
        const bool whole = sh.bucket == need;
        __syncthreads();
        if (whole) break;
    }

    // Compaction: thread owns a contiguous index run [b, e).
    const int per = (n + kSelThreads - 1) / kSelThreads;
    const int b = min(n, static_cast<int>(threadIdx.x) * per), e = min(n, b + per);
    uint32_t n_eq = 0;
    for (int i = b; i < e; ++i) n_eq += (key_at(i) & mask) == prefix;
    uint32_t tot;
    uint32_t eq_rank = block_exclusive_scan(n_eq, sh.warp, &tot);
    uint32_t n_sel = 0;
    {
        uint32_t r = eq_rank;
        for (int i = b; i < e; ++i) {
            const uint64_t km = key_at(i) & mask;
            if (km > prefix) ++n_sel;
            else if (km == prefix) n_sel += (r++ < need);
        }
    }
    uint32_t pos = block_exclusive_scan(n_sel, sh.warp, &tot);
    for (int i = b; i < e; ++i) {
        const uint64_t km = key_at(i) & mask;
        bool take = km > prefix;
        if (km == prefix) take = eq_rank++ < need;
        if (take) out[static_cast<int64_t>(pos++) * heads] = static_cast<uint32_t>(i);
    }
}

// Register-resident variant for segments of up to 16 * 1024 scores (every configuration of the path): thread t owns
// the KPT contiguous indices [t*KPT, t*KPT + KPT) and keeps their keys in registers through every pass, so HBM is
// read once (all loads issued back to back).  The radix starts below the common prefix of the segment's minimum and
// maximum key (one block reduction), which both skips the passes that cannot discriminate (sign / exponent bits
// shared by all scores) and spreads the first histogram — shared-memory atomics then rarely collide.
constexpr int kRegThreads = 1024;
constexpr int kRegWarps = kRegThreads / 32;

struct RegShared {
    uint32_t hist[256];
    uint32_t warp[kRegWarps];
    uint64_t red[kRegWarps];
    uint64_t prefix;
    uint32_t need;
    uint32_t bucket;
};

__device__ __forceinline__ uint32_t block_scan_1024(uint32_t v, uint32_t* warp_sums, uint32_t* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += x;
    }
    if (lane == 31) warp_sums[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        uint32_t w = warp_sums[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t x = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += x;
        }
        warp_sums[lane] = w;
    }
    __syncthreads();
    const uint32_t before = wid ? warp_sums[wid - 1] : 0u;
    *total = warp_sums[kRegWarps - 1];
    __syncthreads();
    return before + incl - v;
}

template <bool kMax>
__device__ __forceinline__ uint64_t block_reduce_u64(uint64_t v, uint64_t* red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t x = __shfl_xor_sync(0xffffffffu, v, o);
        v = kMax ? (x > v ? x : v) : (x < v ? x : v);
    }
    if (lane == 0) red[wid] = v;
    __syncthreads();
    v = red[lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t x = __shfl_xor_sync(0xffffffffu, v, o);
        v = kMax ? (x > v ? x : v) : (x < v ? x : v);
    }
    __syncthreads();
    return v;
}

template <int KPT>
__global__ void __launch_bounds__(kRegThreads) select_reg_kernel(const double* __restrict__ scores,
                                                                 const int64_t* __restrict__ tok_off,
                                                                 const int64_t* __restrict__ keep,
                                                                 const int64_t* __restrict__ row_off, int heads,
                                                                 uint32_t* __restrict__ idx_out) {
    __shared__ RegShared sh;
    const int g = blockIdx.x / heads;
    const int h = blockIdx.x - g * heads;
    const int64_t t0 = tok_off[g];
    const int n = static_cast<int>(tok_off[g + 1] - t0);
    const double* s = scores + heads * t0 + static_cast<int64_t>(h) * n;
    const int64_t kk = keep[g];
    const int k = kk < n ? static_cast<int>(kk) : n;
    uint32_t* out = idx_out + row_off[g] * heads + h;
    if (k <= 0) return;
    if (k == n) {  // everything kept, in order
        for (int i = threadIdx.x; i < n; i += kRegThreads) out[static_cast<int64_t>(i) * heads] = i;
        return;
    }
    const int base = static_cast<int>(threadIdx.x) * KPT;
    uint64_t key[KPT];
#pragma unroll
    for (int e = 0; e < KPT; ++e) key[e] = base + e < n ? score_key(__ldg(s + base + e)) : 0ull;
    uint64_t lo = ~0ull, hi = 0;
#pragma unroll
    for (int e = 0; e < KPT; ++e) {
        if (base + e < n) {
            lo = key[e] < lo ? key[e] : lo;
            hi = key[e] > hi ? key[e] : hi;
        }
    }
    lo = block_reduce_u64<false>(lo, sh.red);
    hi = block_reduce_u64<true>(hi, sh.red);

    // Threshold bucket: keys whose bits above `bit` equal `prefix` (mask); `need` of them are still to be taken.
    uint64_t mask = 0, prefix = 0;
    uint32_t need = static_cast<uint32_t>(k);
    if (lo != hi) {
        int top = 63 - __clzll(static_cast<long long>(lo ^ hi));  // highest bit in which the keys differ
        mask = top == 63 ? 0ull : ~((2ull << top) - 1);
        prefix = lo & mask;
        while (top >= 0) {
            const int width = top >= 7 ? 8 : top + 1;
            const int shift = top - width + 1;
            const uint32_t dmask = (1u << width) - 1;
            if (threadIdx.x < 256) sh.hist[threadIdx.x] = 0;
            __syncthreads();
#pragma unroll
            for (int e = 0; e < KPT; ++e)
                if (base + e < n && (key[e] & mask) == prefix)
                    atomicAdd(&sh.hist[static_cast<uint32_t>(key[e] >> shift) & dmask], 1u);
            __syncthreads();
            // suffix scan over the bins (largest digit first): thread b < 256 looks at digit 255 - b
            uint32_t c = threadIdx.x < 256 ? sh.hist[255 - threadIdx.x] : 0u;
            uint32_t tot;
            const uint32_t excl = block_scan_1024(c, sh.warp, &tot);
            if (threadIdx.x < 256 && excl < need && excl + c >= need) {
                sh.prefix = prefix | (static_cast<uint64_t>(255 - threadIdx.x) << shift);
                sh.need = need - excl;
                sh.bucket = c;
            }
            __syncthreads();
            prefix = sh.prefix;
            need = sh.need;
            mask |= static_cast<uint64_t>(dmask) << shift;
            const bool whole = sh.bucket == need;
            __syncthreads();
            if (whole) break;
            top = shift - 1;
        }
    }
    // else: every key equal — the first k indices (index tie-break), i.e. all keys in the bucket, first `need`.

    // Ascending compaction: keys above the bucket are all taken; bucket keys by index rank < need.
    uint32_t n_eq = 0, n_gt = 0;
#pragma unroll
    for (int e = 0; e < KPT; ++e) {
        if (base + e < n) {
            const uint64_t km = key[e] & mask;
            n_eq += km == prefix;
            n_gt += km > prefix;
        }
    }
    uint32_t tot;
    uint32_t eq_rank = block_scan_1024(n_eq, sh.warp, &tot);
    const uint32_t n_take_eq = eq_rank >= need ? 0u : (need - eq_rank < n_eq ? need - eq_rank : n_eq);
    uint32_t pos = block_scan_1024(n_gt + n_take_eq, sh.warp, &tot);
#pragma unroll
    for (int e = 0; e < KPT; ++e) {
        if (base + e < n) {
            const uint64_t km = key[e] & mask;
            bool take = km > prefix;
            if (km == prefix) take = eq_rank++ < need;
            if (take) out[static_cast<int64_t>(pos++) * heads] = static_cast<uint32_t>(base + e);
        }
    }
}

}  // namespace

int launch_select(cudaStream_t stream, const qvk_groups* g, const double* scores, int heads, uint32_t* idx) {
    const int64_t segs = static_cast<int64_t>(g->n_groups) * heads;
    if (segs == 0) return QVK_OK;
    if (segs > 0x7fffffff) QVK_INVALID("select: too many segments");
    auto reg = [&](auto kern) {
        kern<<<static_cast<unsigned>(segs), kRegThreads, 0, stream>>>(scores, g->tok_off_d, g->keep_d, g->row_off_d,
                                                                      heads, idx);
        QVK_LAUNCH_CHECK();
        return QVK_OK;
    };
    if (g->max_tokens <= 1 * kRegThreads) return reg(select_reg_kernel<1>);
    if (g->max_tokens <= 2 * kRegThreads) return reg(select_reg_kernel<2>);
    if (g->max_tokens <= 4 * kRegThreads) return reg(select_reg_kernel<4>);
    if (g->max_tokens <= 8 * kRegThreads) return reg(select_reg_kernel<8>);
    if (g->max_tokens <= 16 * kRegThreads) return reg(select_reg_kernel<16>);
    const size_t smem = static_cast<size_t>(g->max_tokens) * sizeof(uint64_t);
    constexpr size_t kMaxDyn = 200 * 1024;
    if (smem <= kMaxDyn) {
        QVK_CUDA_CHECK(func_attr(reinterpret_cast<const void*>(select_kernel<true>),
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kMaxDyn)));
        select_kernel<true><<<static_cast<unsigned>(segs), kSelThreads, smem, stream>>>(
            scores, g->tok_off_d, g->keep_d, g->row_off_d, heads, idx);
    } else {
        select_kernel<false><<<static_cast<unsigned>(segs), kSelThreads, 0, stream>>>(
            scores, g->tok_off_d, g->keep_d, g->row_off_d, heads, idx);
    }
    QVK_LAUNCH_CHECK();
    return QVK_OK;
}

}  // namespace qvk
