// (a5)+(a9)+(a10) fused prune: score -> top-k -> KV compaction for every (group, head) segment in ONE launch.
//
// prune_group (prefill.cpp:255-282) is three dependent steps; as three kernels (score.cu, select.cu, gather.cu) the
// select step is latency-bound (one CTA per segment, 2.6 MB of algorithmic traffic) and every launch pays its own
// ramp and tail.  Here a THREAD-BLOCK CLUSTER of CL CTAs (CL = 1..16, about 1024 rows per CTA) owns one segment
// (N_g rows of one head of one group):
//   1. score: CTA c scores rows [c*R, (c+1)*R) (R = ceil(N_g / CL)) straight from HBM — a row (width bf16) is read
//      by W/32 lanes with 4 x 16-byte loads each, two rows in flight per lane group; bf16 magnitudes become doubles
//      with integer ops (no F2F) — and keeps the double scores of its rows in shared memory.  Scores are bit-identical to the reference
//      (prefill.cpp:207: the order-free double sum is exact whenever the row passes the exactness test of
//      score.cu; the rare rows that fail it are re-summed in the reference's sequential order).
//      With kScore = false the scores come from HBM instead (SnapKV, snapkv.cu).
//   2. select: MSB-first radix select over the whole segment — every CTA builds the 256-bin histogram of its own
//      keys, the cluster sums the CL histograms through distributed shared memory (mapa +
//      ld.shared::cluster), and every CTA picks the same digit, so the threshold is agreed without HBM traffic.
//      Starts below the common prefix of the segment's min / max key and stops once the threshold bucket is taken
//      whole (same rounds as select_reg_kernel, select.cu).
//   3. compaction: index order within the segment = (CTA rank, local row), so one exchange of per-CTA counts gives
//      each CTA its output base; then the CTA copies its retained K and V rows (K mostly from L2: it was read in
//      step 1) to the cache with coalesced 16-byte stores, plus idx and origin (prefill.cpp:277-280, 304-308).
// Result identical to score -> nth_element + sort under (score desc, index asc), -0.0 == +0.0 -> ascending gather.
// Algorithmic bytes per (group, head): N*W*2 (scored tensor) + k*(W*2 (other tensor) + 2*W*2 (writes) + 8 + 4)
// + N*8 (scores, when written).
#include <cstdlib>

#include "common.cuh"
#include "ptx.cuh"

namespace qvk {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxRowsPerCta = 4096;
constexpr int kRowsTarget = 1024;  // rows per CTA the cluster size aims for (measured best of 256..4096)

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t dsmem_addr(const void* p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(ptx::smem_u32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ uint32_t ld_dsmem_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t ld_dsmem_u64(uint32_t a) {
    uint64_t v;
    asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_sync() {
    cluster_arrive();
    cluster_wait();
}

#ifdef QVK_PRUNE_TRACE
// Developer timeline (tools/prune_trace.cu): %globaltimer_lo at the phase boundaries of every CTA.
__device__ uint32_t* g_prune_trace;
__device__ uint32_t* g_prune_smid;
__device__ __forceinline__ void prune_trace(int slot) {
    if (threadIdx.x == 0) {
        uint32_t t;
        asm volatile("mov.u32 %0, %%globaltimer_lo;" : "=r"(t));
        g_prune_trace[blockIdx.x * 8 + slot] = t;
        if (slot == 0) {
            uint32_t sm;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
            g_prune_smid[blockIdx.x] = sm;
        }
    }
}
#define QVK_PT(slot) prune_trace(slot)
#else
#define QVK_PT(slot)
#endif

// Cache destinations of the compaction: dest 0 is this GPU's cache; dests 1..n-1 are the same cache buffers of the
// other ranks, mapped into this process over NVLink (CUDA IPC peer pointers, distributed.py PeerCache) — the
// all-gather of the pruned rows fused into the gather (each retained row is read once and stored n times).
constexpr int kMaxDests = 8;
struct Dests {
    int n;
    __nv_bfloat16* kc[kMaxDests];
    __nv_bfloat16* vc[kMaxDests];
    uint64_t* org[kMaxDests];
};

struct FusedShared {
    uint32_t hist[2][256];  // double-buffered: round r writes hist[r & 1] (one cluster barrier per round)
    uint32_t warp[kWarps];
    uint64_t red[kWarps];
    uint64_t lo, hi;        // this CTA's min / max key (published to the cluster)
    uint32_t cnt[256];      // cluster-summed histogram, suffix order
    uint32_t n_tot;         // this CTA's (gt << 16 | eq) counts at the threshold (published)
    uint64_t prefix;
    uint32_t need, bucket;
};

__device__ __forceinline__ uint32_t block_scan(uint32_t v, uint32_t* warp_sums, uint32_t* total) {
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
        uint32_t w = lane < kWarps ? warp_sums[lane] : 0u;
#pragma unroll
        for (int o = 1; o < kWarps; o <<= 1) {
            const uint32_t x = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += x;
        }
        if (lane < kWarps) warp_sums[lane] = w;
    }
    __syncthreads();
    const uint32_t before = wid ? warp_sums[wid - 1] : 0u;
    *total = warp_sums[kWarps - 1];
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
    v = red[0];
#pragma unroll
    for (int w = 1; w < kWarps; ++w) v = kMax ? (red[w] > v ? red[w] : v) : (red[w] < v ? red[w] : v);
    __syncthreads();
    return v;
}

// Reference-order (prefill.cpp:207) sum of squares of a bf16 row in HBM: the rare fallback of the exact test.
__device__ __noinline__ double seq_sumsq_global(const uint4* row, int chunks) {
    double acc = 0.0;
    for (int c = 0; c < chunks; ++c) {
        const uint4 p = __ldg(row + c);
        const uint32_t w[4] = {p.x, p.y, p.z, p.w};
        for (int e = 0; e < 8; ++e) {
            const uint32_t bits = (e & 1) ? (w[e >> 1] & 0xffff0000u) : (w[e >> 1] << 16);
            const double d = static_cast<double>(__uint_as_float(bits));
            acc = __fma_rn(d, d, acc);  // d*d is exact for bf16, so this rounds like acc + d*d
        }
    }
    return acc;
}


// W = row width in bf16 elements (64..512); CL = CTAs per segment (cluster size); kScore: compute norm scores
// (negate = key_norm_small) from x, else read the double scores (SnapKV).
template <int W, int CL, bool kScore>
__global__ void __launch_bounds__(kThreads) prune_fused_kernel(
    const __nv_bfloat16* __restrict__ x, const double* __restrict__ scores_in, int negate,
    const __nv_bfloat16* __restrict__ k, const __nv_bfloat16* __restrict__ v, int heads,
    const int64_t* __restrict__ tok_off, const int64_t* __restrict__ keep, const int64_t* __restrict__ row_off,
    const uint64_t* __restrict__ first_token, double* __restrict__ scores_out, uint32_t* __restrict__ idx_out,
    const Dests dst, int overlap_prev) {
    constexpr int kChunks = W / 8;     // 16-byte chunks per row
    constexpr int kCpl = 4;            // 16-byte chunks per lane per row (chunk sl + c*kLpr)
    constexpr int kLpr = kChunks / kCpl;  // lanes per row: 2 / 4 / 8 / 16
    constexpr int kRpp = kThreads / kLpr;  // rows per pass
    static_assert(kChunks % kCpl == 0 && kLpr >= 2 && kLpr <= 32, "width");
    extern __shared__ double sc[];  // [R] this CTA's scores (doubles), then [R] u16 selected local rows
    __shared__ FusedShared sh;

    const uint32_t crank = CL > 1 ? cluster_rank() : 0u;
    // PDL (launched with programmatic stream serialization).  Default: wait here for the previous kernel, which may
    // have produced K / V.  overlap_prev: the previous kernel is independent of our inputs (qvk_prefill_layer's
    // attention, which only reads K / V that were complete before it started), so start now and wait at the end
    // instead — our completion still implies the previous kernel's, keeping the stream order for later work.
    if (!overlap_prev) asm volatile("griddepcontrol.wait;" ::: "memory");
    const int64_t seg = blockIdx.x / CL;
    const int g = static_cast<int>(seg / heads);
    const int h = static_cast<int>(seg - static_cast<int64_t>(g) * heads);
    const int64_t t0 = tok_off[g];
    const int n = static_cast<int>(tok_off[g + 1] - t0);
    if (n <= 0) {  // uniform over the cluster
        if (overlap_prev) asm volatile("griddepcontrol.wait;" ::: "memory");
        return;
    }
    const int64_t kk = keep[g];
    const int kseg = kk < n ? static_cast<int>(kk) : n;
    const int R = (n + CL - 1) / CL;
    const int r0 = min(n, static_cast<int>(crank) * R);
    const int nr = min(n, r0 + R) - r0;  // rows of this CTA (may be 0)
    uint16_t* sel = reinterpret_cast<uint16_t*>(sc + R);

    const int tid = threadIdx.x;
    const int slot = tid / kLpr, sl = tid - slot * kLpr;  // row slot in a pass, lane within the row
    QVK_PT(0);
    // ---- 1. scores of this CTA's rows ------------------------------------------------------------------------------
    if constexpr (kScore) {
        // Software pipeline: the loads of pass p + 1 are in flight while pass p is summed.
        auto load = [&](int p0, uint4 (&buf)[kCpl]) {
            const int r = p0 + slot;
            const uint4* row = reinterpret_cast<const uint4*>(x + ((t0 + r0 + r) * heads + h) * W);
#pragma unroll
            for (int c = 0; c < kCpl; ++c) buf[c] = r < nr ? __ldg(row + sl + c * kLpr) : make_uint4(0u, 0u, 0u, 0u);
        };
        auto consume = [&](int p0, const uint4 (&buf)[kCpl]) {
            double acc[2] = {0.0, 0.0};
            uint32_t mn2 = 0xffffffffu, mx2 = 0u;  // per 16-bit half: min(|x| - 1), max |x|
#pragma unroll
            for (int c = 0; c < kCpl; ++c) {
                const uint32_t w[4] = {buf[c].x, buf[c].y, buf[c].z, buf[c].w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t a = w[q] & 0x7fff7fffu;
                    mx2 = __vmaxu2(mx2, a);
                    mn2 = __vminu2(mn2, __vsub2(a, 0x00010001u));
                    const double dl = ptx::bf16_lo_scaled(w[q]), dh = ptx::bf16_hi_scaled(w[q]);
                    acc[0] = __fma_rn(dl, dl, acc[0]);  // squares of bf16 values are exact in double
                    acc[1] = __fma_rn(dh, dh, acc[1]);
                }
            }
            double sum = __dadd_rn(acc[0], acc[1]);
            uint32_t mn = min(mn2 & 0xffffu, mn2 >> 16), mx = max(mx2 & 0xffffu, mx2 >> 16);
#pragma unroll
            for (int o = 1; o < kLpr; o <<= 1) {
                sum = __dadd_rn(sum, __shfl_xor_sync(0xffffffffu, sum, o));
                mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
                mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            }
            // Exactness (score.cu): every square is a multiple of 2^q, q = 2 (E_min - 134); if the total is below
            // 2^(q + 53) every partial sum of any order is exact == the reference's sequential sum.  Subnormals
            // (0 < |x| < 0x80) and inf / nan (|x| >= 0x7f80) are not representable above: sequential fallback.
            bool exact = mx < 0x7f80u;
            if (mn != 0xffffu) {  // some nonzero element: mn + 1 = smallest nonzero magnitude
                exact = exact && mn + 1 >= (37u << 7);  // >= 2^-90: the zero elements' stand-ins are absorbed
                const int qmin = 2 * (static_cast<int>((mn + 1) >> 7) - 134);
                const int es = static_cast<int>((__double_as_longlong(sum) >> 52) & 0x7ff) - 1023 - 256;
                exact = exact && es <= qmin + 52;
                sum *= 0x1p-256;  // unscale (exact: the sum is >= 2^-180)
            } else {
                sum = 0.0;  // all zero
            }
            const int r = p0 + slot;
            if (sl == 0 && r < nr) {
                if (!exact)
                    sum = seq_sumsq_global(reinterpret_cast<const uint4*>(x + ((t0 + r0 + r) * heads + h) * W),
                                           kChunks);
                const double norm = __dsqrt_rn(sum);
                sc[r] = negate ? -norm : norm;  // zero row -> -0.0 like the reference
            }
        };
        uint4 bufa[kCpl], bufb[kCpl];
        if (nr > 0) load(0, bufa);
        for (int p0 = 0; p0 < nr; p0 += 2 * kRpp) {
            if (p0 + kRpp < nr) load(p0 + kRpp, bufb);
            consume(p0, bufa);
            if (p0 + kRpp >= nr) break;
            if (p0 + 2 * kRpp < nr) load(p0 + 2 * kRpp, bufa);
            consume(p0 + kRpp, bufb);
        }
    } else {
        const double* s = scores_in + heads * t0 + static_cast<int64_t>(h) * n + r0;
        for (int r = tid; r < nr; r += kThreads) sc[r] = __ldg(s + r);
    }
    __syncthreads();
    QVK_PT(1);
    uint64_t lo = ~0ull, hi = 0ull;
    for (int r = tid; r < nr; r += kThreads) {
        const uint64_t key = score_key(sc[r]);
        lo = key < lo ? key : lo;
        hi = key > hi ? key : hi;
    }
    lo = block_reduce_u64<false>(lo, sh.red);
    hi = block_reduce_u64<true>(hi, sh.red);
    if constexpr (CL > 1) {
        if (tid == 0) {
            sh.lo = lo;
            sh.hi = hi;
        }
        cluster_sync();  // lo / hi published (CTAs without rows publish the neutral (~0, 0))
        lo = ~0ull;
        hi = 0ull;
#pragma unroll
        for (int c = 0; c < CL; ++c) {
            const uint64_t a = ld_dsmem_u64(dsmem_addr(&sh.lo, c)), b = ld_dsmem_u64(dsmem_addr(&sh.hi, c));
            lo = a < lo ? a : lo;
            hi = b > hi ? b : hi;
        }
    }

    QVK_PT(2);
    // ---- 2. cluster radix select: threshold bucket = keys with (key & mask) == prefix, `need` of them taken ------
    uint64_t mask = 0, prefix = 0;
    uint32_t need = static_cast<uint32_t>(kseg);
    if (kseg < n && lo != hi) {
        int top = 63 - __clzll(static_cast<long long>(lo ^ hi));
        mask = top == 63 ? 0ull : ~((2ull << top) - 1);
        prefix = lo & mask;
        int round = 0;
        while (top >= 0) {
            const int wd = top >= 7 ? 8 : top + 1;
            const int shift = top - wd + 1;
            const uint32_t dmask = (1u << wd) - 1;
            uint32_t* hist = sh.hist[round & 1];
            hist[tid] = 0;  // kThreads == 256 bins
            __syncthreads();
            for (int r = tid; r < nr; r += kThreads) {
                const uint64_t key = score_key(sc[r]);
                if ((key & mask) == prefix) atomicAdd(&hist[static_cast<uint32_t>(key >> shift) & dmask], 1u);
            }
            uint32_t c = 0;
            if constexpr (CL > 1) {
                cluster_sync();  // every CTA's histogram complete
#pragma unroll
                for (int q = 0; q < CL; ++q) c += ld_dsmem_u32(dsmem_addr(&hist[255 - tid], q));
            } else {
                __syncthreads();
                c = hist[255 - tid];
            }
            // position p = tid holds digit 255 - p (suffix order); one warp scans the 256 positions, 8 per lane
            sh.cnt[tid] = c;
            __syncthreads();
            if (tid < 32) {
                uint32_t cv[8], sum = 0;
#pragma unroll
                for (int i = 0; i < 8; ++i) sum += (cv[i] = sh.cnt[tid * 8 + i]);
                uint32_t incl = sum;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (tid >= o) incl += y;
                }
                uint32_t run = incl - sum;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    if (run < need && run + cv[i] >= need) {
                        sh.prefix = prefix | (static_cast<uint64_t>(255 - (tid * 8 + i)) << shift);
                        sh.need = need - run;
                        sh.bucket = cv[i];
                    }
                    run += cv[i];
                }
            }
            __syncthreads();
            prefix = sh.prefix;  // sh.* is rewritten only after the next round's barriers
            need = sh.need;
            mask |= static_cast<uint64_t>(dmask) << shift;
            const bool whole = sh.bucket == need;
            ++round;
            if (whole) break;
            top = shift - 1;
        }
#ifdef QVK_PRUNE_TRACE
        if (threadIdx.x == 0) g_prune_smid[blockIdx.x] |= static_cast<uint32_t>(round) << 16;
#endif
    }
    // else: every key equal, or k == N: mask = 0 puts all keys in the bucket, the first `need` (= k) by index.

    QVK_PT(3);
    // ---- 3. compaction: thread owns contiguous local rows [b, e) ----------------------------------------------------
    const int per = (nr + kThreads - 1) / kThreads;
    const int b = min(nr, tid * per), e = min(nr, b + per);
    uint32_t n_eq = 0, n_gt = 0;
    for (int i = b; i < e; ++i) {
        const uint64_t km = score_key(sc[i]) & mask;
        n_eq += km == prefix;
        n_gt += km > prefix;
    }
    uint32_t cta_tot;  // packed (gt << 16 | eq): R <= 4096 rows per CTA
    const uint32_t before = block_scan((n_gt << 16) | n_eq, sh.warp, &cta_tot);
    const uint32_t eq_local = before & 0xffffu, gt_local = before >> 16;
    uint32_t eq_base = 0, out_base = 0;  // equal keys / output rows before this CTA (lower ranks first)
    if constexpr (CL > 1) {
        if (tid == 0) sh.n_tot = cta_tot;
        cluster_sync();
        for (uint32_t c = 0; c < crank; ++c) {
            const uint32_t t = ld_dsmem_u32(dsmem_addr(&sh.n_tot, c));
            const uint32_t ce = t & 0xffffu;
            out_base += (t >> 16) + (eq_base >= need ? 0u : min(need - eq_base, ce));
            eq_base += ce;
        }
        cluster_arrive();  // last remote read done; the matching wait precedes exit (peers read our smem)
    }
    // equal keys are taken in index order while the segment-wide equal rank is below `need`
    const uint32_t eq_quota = need > eq_base ? need - eq_base : 0u;
    const uint32_t cta_sel = (cta_tot >> 16) + min(eq_quota, cta_tot & 0xffffu);
    uint32_t eq_rank = eq_base + eq_local;
    uint32_t pos = gt_local + min(eq_quota, eq_local);
    for (int i = b; i < e; ++i) {
        const uint64_t km = score_key(sc[i]) & mask;
        bool take = km > prefix;
        if (km == prefix) take = eq_rank++ < need;
        if (take) sel[pos++] = static_cast<uint16_t>(i);
    }
    __syncthreads();

    QVK_PT(4);
    // ---- gather the selected rows: K, V -> cache, idx, origin; then the scores (coalesced) ----------------------
    const int64_t crow0 = row_off[g] + out_base;  // cache row of this CTA's first selected row
    const uint64_t ft = first_token ? first_token[g] : 0ull;
    const int nsel = static_cast<int>(cta_sel);
    for (int s0 = 0; s0 < nsel; s0 += kRpp) {
        const int s = s0 + slot;
        if (s < nsel) {
            const int j = sel[s];
            const int64_t src = ((t0 + r0 + j) * heads + h) * W;
            uint4 bk[kCpl], bv[kCpl];
#pragma unroll
            for (int c = 0; c < kCpl; ++c) {
                bk[c] = __ldg(reinterpret_cast<const uint4*>(k + src) + sl + c * kLpr);
                bv[c] = __ldg(reinterpret_cast<const uint4*>(v + src) + sl + c * kLpr);
            }
            const int64_t cu = (crow0 + s) * heads + h;  // cache unit
            const uint32_t jj = static_cast<uint32_t>(r0 + j);
            for (int dd = 0; dd < dst.n; ++dd) {
#pragma unroll
                for (int c = 0; c < kCpl; ++c) {
                    reinterpret_cast<uint4*>(dst.kc[dd] + cu * W)[sl + c * kLpr] = bk[c];
                    reinterpret_cast<uint4*>(dst.vc[dd] + cu * W)[sl + c * kLpr] = bv[c];
                }
                if (sl == 0 && dst.org[dd]) dst.org[dd][cu] = ft + jj;
            }
            if (sl == 0 && idx_out) idx_out[cu] = jj;
        }
    }
    if (dst.n > 1) __threadfence_system();  // peer stores visible system-wide before the kernel's completion
    QVK_PT(5);
    if (kScore && scores_out) {
        double* so = scores_out + heads * t0 + static_cast<int64_t>(h) * n + r0;
        for (int r = tid; r < nr; r += kThreads) so[r] = sc[r];
    }
    QVK_PT(6);
    if constexpr (CL > 1) cluster_wait();
    if (overlap_prev) asm volatile("griddepcontrol.wait;" ::: "memory");
    QVK_PT(7);
}

template <int W, int CL, bool kScore>
int launch_wc(cudaStream_t stream, const qvk_groups* g, const void* x, const double* scores_in, int negate,
              const void* k, const void* v, int heads, double* scores_out, uint32_t* idx, const Dests& dst,
              int overlap_prev) {
    const int64_t segs = static_cast<int64_t>(g->n_groups) * heads;
    const int rmax = static_cast<int>((g->max_tokens + CL - 1) / CL);
    const size_t smem = static_cast<size_t>(rmax) * (sizeof(double) + sizeof(uint16_t)) + 16;
    auto kern = prune_fused_kernel<W, CL, kScore>;
    if (CL > 8)
        QVK_CUDA_CHECK(func_attr(reinterpret_cast<const void*>(kern), cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    if (smem > 48 * 1024)
        QVK_CUDA_CHECK(func_attr(reinterpret_cast<const void*>(kern), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(segs * CL));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // overlap the launch with the previous kernel
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    QVK_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, static_cast<const __nv_bfloat16*>(x), scores_in, negate,
                                      static_cast<const __nv_bfloat16*>(k), static_cast<const __nv_bfloat16*>(v),
                                      heads, g->tok_off_d, g->keep_d, g->row_off_d, g->first_token_d, scores_out,
                                      idx, dst, overlap_prev));
    return QVK_OK;
}

// Cluster size: about kRowsTarget rows per CTA, doubled (up to 16) while the grid would leave SMs idle.  Scoring
// launches (which stream every K row) double until ~2 CTAs per SM when there are fewer segments than SMs (C2: 64
// segments -> 8-CTA clusters, 54 us; one CTA per SM: 56 us); otherwise — and always for select + gather on given
// scores, where the cluster exchanges outweigh the smaller streams — only until every SM has a CTA (C3: 256
// segments of 1024 rows stay 1 CTA each, select + gather 24.6 vs 30.7 us with 2-CTA clusters; C2 select + gather
// 38.9 vs 49.2 us with 4- instead of 16-CTA clusters).
int cluster_size(int64_t segs, int64_t max_tokens, bool score) {
    // tuning knobs QVK_PRUNE_ROWS (rows per CTA), QVK_PRUNE_FILL (CTAs per SM of scoring launches, segments < SMs)
    static const int target = std::max(64, env_knob("QVK_PRUNE_ROWS", kRowsTarget));
    static const int fill_small = std::max(1, env_knob("QVK_PRUNE_FILL", 2));
    const int fill = score && segs < kNumSms ? fill_small : 1;
    int cl = 1;
    while (cl < 16 && max_tokens > static_cast<int64_t>(cl) * target) cl *= 2;
    while (cl < 16 && segs * cl < fill * kNumSms && max_tokens >= static_cast<int64_t>(cl) * 2 * 128) cl *= 2;
    return cl;
}

template <int W, bool kScore>
int launch_w(cudaStream_t stream, const qvk_groups* g, const void* x, const double* scores_in, int negate,
             const void* k, const void* v, int heads, double* scores_out, uint32_t* idx, const Dests& dst,
             int ov) {
    switch (cluster_size(static_cast<int64_t>(g->n_groups) * heads, g->max_tokens, kScore)) {
        case 1: return launch_wc<W, 1, kScore>(stream, g, x, scores_in, negate, k, v, heads, scores_out, idx, dst, ov);
        case 2: return launch_wc<W, 2, kScore>(stream, g, x, scores_in, negate, k, v, heads, scores_out, idx, dst, ov);
        case 4: return launch_wc<W, 4, kScore>(stream, g, x, scores_in, negate, k, v, heads, scores_out, idx, dst, ov);
        case 8: return launch_wc<W, 8, kScore>(stream, g, x, scores_in, negate, k, v, heads, scores_out, idx, dst, ov);
        default: return launch_wc<W, 16, kScore>(stream, g, x, scores_in, negate, k, v, heads, scores_out, idx, dst, ov);
    }
}

}  // namespace

// True when the fused kernel covers this shape: bf16 rows of 64..512 elements (multiple of 64), 16-byte aligned
// tensors, segments of at most kCluster * kMaxRowsPerCta rows.
bool prune_fused_supported(const qvk_groups* g, int dtype, int width, const void* k, const void* v, const void* kc,
                           const void* vc) {
    const uintptr_t al = reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v) |
                         reinterpret_cast<uintptr_t>(kc) | reinterpret_cast<uintptr_t>(vc);
    return dtype == QVK_BF16 && (width == 64 || width == 128 || width == 256 || width == 512) && (al & 15) == 0 &&
           g->max_tokens <= 16 * static_cast<int64_t>(kMaxRowsPerCta) &&
           static_cast<int64_t>(g->n_groups) * 16 < (int64_t(1) << 31) / 8;
}

// Per-token pruning (heads == 1, the reference's own semantics) of a small batch lands on 16-CTA clusters, which lose
// to the three separate kernels (16 x 4096 tokens, width 512: 83 vs 60 us; width 256: 49 vs 42 us); from ~32
// segments on the fused launch wins (225 x 4096, width 512: 510 vs 552 us).  Knob QVK_PRUNE_FUSED_MIN_SEGS.
bool prune_fused_preferred(const qvk_groups* g, int heads) {
    static const int min_segs = std::max(0, env_knob("QVK_PRUNE_FUSED_MIN_SEGS", 32));
    return !(heads == 1 && static_cast<int64_t>(g->n_groups) < min_segs);
}

// scorer: QVK_KEY_NORM_SMALL / QVK_VALUE_NORM (scores computed here; written to scores_out when non-null) or
// QVK_SNAPKV = any precomputed scores in scores_in (SnapKV, or the key-norm fused into the projection).
// overlap_prev: the previous kernel on `stream` does not produce k / v (see the kernel's PDL note).
// n_dest caches (dest 0 local, the rest peer mappings of the same buffers): the compaction stores every retained row
// into all of them (<= 8).
int launch_prune_fused_dests(cudaStream_t stream, const qvk_groups* g, const void* k, const void* v, int heads,
                             int width, int scorer, const double* scores_in, double* scores_out, uint32_t* idx,
                             int n_dest, void* const* kc, void* const* vc, uint64_t* const* origin,
                             int overlap_prev) {
    if (static_cast<int64_t>(g->n_groups) * heads == 0 || g->max_tokens == 0) return QVK_OK;
    if (n_dest < 1 || n_dest > kMaxDests) QVK_INVALID("prune: 1..8 cache destinations");
    if (origin && !g->first_token_d)
        for (int i = 0; i < n_dest; ++i)
            if (origin[i]) QVK_INVALID("gather: origin requested without first_token");
    Dests dst{};
    dst.n = n_dest;
    for (int i = 0; i < n_dest; ++i) {
        dst.kc[i] = static_cast<__nv_bfloat16*>(kc[i]);
        dst.vc[i] = static_cast<__nv_bfloat16*>(vc[i]);
        dst.org[i] = origin ? origin[i] : nullptr;
    }
    const bool pre = scorer == QVK_SNAPKV;
    const void* x = scorer == QVK_VALUE_NORM ? v : k;
    const int negate = scorer == QVK_KEY_NORM_SMALL;
#define QVK_FUSED_CASE(WW)                                                                                        \
    case WW:                                                                                                      \
        return pre ? launch_w<WW, false>(stream, g, x, scores_in, negate, k, v, heads, nullptr, idx, dst,         \
                                         overlap_prev)                                                            \
                   : launch_w<WW, true>(stream, g, x, nullptr, negate, k, v, heads, scores_out, idx, dst,         \
                                        overlap_prev);
    switch (width) {
        QVK_FUSED_CASE(64)
        QVK_FUSED_CASE(128)
        QVK_FUSED_CASE(256)
        QVK_FUSED_CASE(512)
        default:
            QVK_INVALID("prune: fused kernel width");
    }
#undef QVK_FUSED_CASE
}

int launch_prune_fused(cudaStream_t stream, const qvk_groups* g, const void* k, const void* v, int heads, int width,
                       int scorer, const double* scores_in, double* scores_out, uint32_t* idx, void* kc, void* vc,
                       uint64_t* origin, int overlap_prev) {
    void* kcs[1] = {kc};
    void* vcs[1] = {vc};
    uint64_t* orgs[1] = {origin};
    return launch_prune_fused_dests(stream, g, k, v, heads, width, scorer, scores_in, scores_out, idx, 1, kcs, vcs,
                                    origin ? orgs : nullptr, overlap_prev);
}

}  // namespace qvk
