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

}  // namespace

int launch_select(cudaStream_t stream, const qvk_groups* g, const double* scores, int heads, uint32_t* idx) {
    const int64_t segs = static_cast<int64_t>(g->n_groups) * heads;
    if (segs == 0) return QVK_OK;
    if (segs > 0x7fffffff) QVK_INVALID("select: too many segments");
    const size_t smem = static_cast<size_t>(g->max_tokens) * sizeof(uint64_t);
    constexpr size_t kMaxDyn = 200 * 1024;
    if (smem <= kMaxDyn) {
        static bool attr_set = false;
        if (!attr_set) {
            QVK_CUDA_CHECK(cudaFuncSetAttribute(select_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                static_cast<int>(kMaxDyn)));
            attr_set = true;
        }
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
