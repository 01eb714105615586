// §8f-4: the consumer of the pruned cache — attention of text / decode query tokens over one layer's compacted K/V
// cache (the step the per-layer all-gather feeds; SPEC.md:380 leaves it as a stub, PAPER.md:221-226 describes the
// pruned cache it reads).
//
//   O[t, h] = softmax_r(scale * q[t, h] . K[r, h / g]) V[r, h / g]   over every cached row r (non-causal: all video
//   tokens precede the queries), g = n_q / n_kv;  LSE[t, h] = ln sum_r exp(scale * q . K[r])  (to merge with the
//   caller's own text-token attention).
//
// HBM-bound for decode (a few query tokens): every cached K/V row must be read once.  Flash-decoding: the rows are
// split into chunks so that (chunks x KV heads x 64-query-row tiles) fills the GPU; a CTA (4 warps, 16 query rows
// each — the g query heads x query tokens sharing one KV head) streams its chunk in 64-row K/V blocks through a
// cp.async double buffer and runs QK^T and PV on the tensor cores (mma.sync m16n8k16 bf16 -> fp32, ldmatrix
// fragments; the operand tiles are too small for tcgen05 and the kernel is memory-bound), online softmax in
// registers; a second kernel merges the chunk partials (max / sum rescaling).
// Algorithmic bytes: 2 * R * n_kv * d * 2 (K and V) + queries and outputs.
#include <cudaTypedefs.h>

#include <cstdlib>

#include "common.cuh"
#include "ptx.cuh"

namespace qvk {
namespace {

constexpr int kDD = 128;           // head dim
constexpr int kQRows = 64;         // query rows per CTA (4 warps x 16)
constexpr int kKvRows = 64;        // cache rows per block
constexpr int kPad = 136;          // smem row stride in elements (272 B: conflict-free ldmatrix)
constexpr int kDecThreads = 128;

struct DecParams {
    const __nv_bfloat16* q;        // (n_tq, n_q, d)
    const __nv_bfloat16* k;        // (rows, n_kv, d)
    const __nv_bfloat16* v;
    int64_t rows;
    int n_tq, n_q, n_kv, group;    // group = n_q / n_kv
    int rows_per_split, splits;
    float scale_log2;
    float* part_o;                 // [n_kv][splits][m_rows][d]
    float* part_ml;                // [n_kv][splits][m_rows][2]  (max in log2 units, sum)
    int m_rows;                    // n_tq * group
};

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], uint32_t addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
        "{%0, %1, %2, %3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool pred) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(pred ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}
__device__ __forceinline__ float ex2f(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// kWS (warp split, m_rows <= 16 — decode of one or two tokens): all four warps share the same 16 query rows and
// take different 16-key quarters of every K/V block, each with its own online-softmax state, written as four
// separate partials (the combine kernel merges them with the chunk partials) — 4x less tensor work per cached row
// than padding the 7 query rows of a KV head to 64.
template <bool kWS>
__global__ void __launch_bounds__(kDecThreads) decode_attention_kernel(const DecParams p) {
    constexpr int kKeys = kWS ? 16 : 64;   // keys of a block each warp processes
    constexpr int kNT = kKeys / 8;         // S n8 tiles per warp
    constexpr int kPVK = kKeys / 16;       // PV k16 steps per warp
    extern __shared__ __align__(16) __nv_bfloat16 sm[];
    __nv_bfloat16* sQ = sm;                          // [64][kPad]
    __nv_bfloat16* sK = sQ + kQRows * kPad;          // [2][64][kPad]
    __nv_bfloat16* sV = sK + 2 * kKvRows * kPad;     // [2][64][kPad]
    const int mtile = blockIdx.x, split = blockIdx.y, h = blockIdx.z;  // m-tiles of one chunk adjacent: L2 reuse
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t r_begin = static_cast<int64_t>(split) * p.rows_per_split;
    const int64_t r_end = min(p.rows, r_begin + p.rows_per_split);
    const int nblocks = static_cast<int>((r_end - r_begin + kKvRows - 1) / kKvRows);

    // Q tile: query row qr = mtile*64 + i -> token qr / group, head h*group + qr % group (zero past m_rows)
    for (int c = tid; c < kQRows * (kDD / 8); c += kDecThreads) {
        const int i = c / (kDD / 8), part = c % (kDD / 8);
        const int qr = mtile * kQRows + i;
        const bool ok = qr < p.m_rows;
        const int t = ok ? qr / p.group : 0, hq = h * p.group + (ok ? qr % p.group : 0);
        cp_async16(static_cast<uint32_t>(__cvta_generic_to_shared(sQ + i * kPad + part * 8)),
                   p.q + (static_cast<int64_t>(t) * p.n_q + hq) * kDD + part * 8, ok);
    }
    auto load_block = [&](int blk, int buf) {
        const int64_t r0 = r_begin + static_cast<int64_t>(blk) * kKvRows;
        for (int c = tid; c < kKvRows * (kDD / 8); c += kDecThreads) {
            const int i = c / (kDD / 8), part = c % (kDD / 8);
            const int64_t r = r0 + i;
            const bool ok = r < r_end;
            const int64_t off = ((ok ? r : 0) * p.n_kv + h) * kDD + part * 8;
            cp_async16(static_cast<uint32_t>(__cvta_generic_to_shared(sK + (buf * kKvRows + i) * kPad + part * 8)),
                       p.k + off, ok);
            cp_async16(static_cast<uint32_t>(__cvta_generic_to_shared(sV + (buf * kKvRows + i) * kPad + part * 8)),
                       p.v + off, ok);
        }
    };
    if (nblocks > 0) load_block(0, 0);
    cp_async_commit();

    const int g = lane >> 2, c4 = lane & 3;
    float o[kDD / 8][4];
#pragma unroll
    for (int i = 0; i < kDD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;  // rows g and g + 8 of the warp's 16
    uint32_t qf[kDD / 16][4];
    bool q_loaded = false;
    const uint32_t sQa = static_cast<uint32_t>(__cvta_generic_to_shared(sQ));
    const uint32_t sKa = static_cast<uint32_t>(__cvta_generic_to_shared(sK));
    const uint32_t sVa = static_cast<uint32_t>(__cvta_generic_to_shared(sV));

    for (int blk = 0; blk < nblocks; ++blk) {
        const int buf = blk & 1;
        if (blk + 1 < nblocks) load_block(blk + 1, buf ^ 1);
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        if (!q_loaded) {
#pragma unroll
            for (int kk = 0; kk < kDD / 16; ++kk) {
                const int row = (kWS ? 0 : warp * 16) + (lane & 7) + 8 * ((lane >> 3) & 1);
                const int col = 16 * kk + 8 * (lane >> 4);
                ldsm_x4(qf[kk], sQa + (row * kPad + col) * 2);
            }
            q_loaded = true;
        }
        // S = Q K^T: 16 rows x kKeys keys per warp (kNT n8 tiles), keys [key0, key0 + kKeys) of the block
        const int key0 = kWS ? 16 * warp : 0;
        float s[kNT][4];
#pragma unroll
        for (int j = 0; j < kNT; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
        for (int kk = 0; kk < kDD / 16; ++kk) {
#pragma unroll
            for (int j = 0; j < kNT; j += 2) {
                uint32_t b[4];
                const int key = key0 + 8 * j + (lane & 7) + 8 * (lane >> 4);
                const int col = 16 * kk + 8 * ((lane >> 3) & 1);
                ldsm_x4(b, sKa + ((buf * kKvRows + key) * kPad + col) * 2);
                mma16816(s[j], qf[kk], b[0], b[1]);
                mma16816(s[j + 1], qf[kk], b[2], b[3]);
            }
        }
        // mask rows past the chunk end, then online softmax (log2 domain)
        const int64_t r0 = r_begin + static_cast<int64_t>(blk) * kKvRows;
        const int valid = static_cast<int>(r_end - r0 < kKvRows ? r_end - r0 : kKvRows);
        float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
        for (int j = 0; j < kNT; ++j)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int key = key0 + 8 * j + 2 * c4 + (e & 1);
                float x = key < valid ? s[j][e] * p.scale_log2 : -INFINITY;
                s[j][e] = x;
                if (e < 2) mx0 = fmaxf(mx0, x);
                else mx1 = fmaxf(mx1, x);
            }
#pragma unroll
        for (int off = 1; off < 4; off <<= 1) {
            mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
            mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
        }
        const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
        const float a0 = mn0 == -INFINITY ? 1.f : ex2f(m0 - mn0), a1 = mn1 == -INFINITY ? 1.f : ex2f(m1 - mn1);
        m0 = mn0;
        m1 = mn1;
        float ps0 = 0.f, ps1 = 0.f;
        uint32_t pf[kPVK][4];  // P as A fragments of the k16 steps of PV
#pragma unroll
        for (int j = 0; j < kNT; ++j) {
            const float p0 = mn0 == -INFINITY ? 0.f : ex2f(s[j][0] - mn0);
            const float p1 = mn0 == -INFINITY ? 0.f : ex2f(s[j][1] - mn0);
            const float p2 = mn1 == -INFINITY ? 0.f : ex2f(s[j][2] - mn1);
            const float p3 = mn1 == -INFINITY ? 0.f : ex2f(s[j][3] - mn1);
            ps0 += p0 + p1;
            ps1 += p2 + p3;
            pf[j >> 1][(j & 1) * 2 + 0] = pack2(p0, p1);
            pf[j >> 1][(j & 1) * 2 + 1] = pack2(p2, p3);
        }
        l0 = l0 * a0 + ps0;
        l1 = l1 * a1 + ps1;
#pragma unroll
        for (int i = 0; i < kDD / 8; ++i) {
            o[i][0] *= a0;
            o[i][1] *= a0;
            o[i][2] *= a1;
            o[i][3] *= a1;
        }
        // O += P V: k = kKeys keys (kPVK steps), n = 128 d (16 n8 tiles)
#pragma unroll
        for (int kk = 0; kk < kPVK; ++kk) {
            // A fragment order: a0 (row g, keys 16kk+2c), a1 (row g+8, same keys), a2 (row g, keys +8), a3 (row g+8)
            const uint32_t a[4] = {pf[kk][0], pf[kk][1], pf[kk][2], pf[kk][3]};
#pragma unroll
            for (int jd = 0; jd < kDD / 8; jd += 2) {
                uint32_t b[4];
                const int key = key0 + 16 * kk + (lane & 7) + 8 * ((lane >> 3) & 1);
                const int col = 8 * jd + 8 * (lane >> 4);
                ldsm_x4_t(b, sVa + ((buf * kKvRows + key) * kPad + col) * 2);
                mma16816(o[jd], a, b[0], b[1]);
                mma16816(o[jd + 1], a, b[2], b[3]);
            }
        }
        __syncthreads();  // buffer `buf` is reloaded by the next iteration's prefetch
    }
    // row sums across the quad, then the partial results of this chunk
#pragma unroll
    for (int off = 1; off < 4; off <<= 1) {
        l0 += __shfl_xor_sync(0xffffffffu, l0, off);
        l1 += __shfl_xor_sync(0xffffffffu, l1, off);
    }
    if constexpr (kWS) {
        // merge the four warps' key quarters in shared memory (the K/V buffers are free now): one partial per CTA
        __syncthreads();
        float* so = reinterpret_cast<float*>(sK);        // [4 warps][16 rows][kDD]
        float* sml = so + 4 * 16 * kDD;                  // [4 warps][16 rows][2]
#pragma unroll
        for (int i = 0; i < kDD / 8; ++i) {
            *reinterpret_cast<float2*>(so + (warp * 16 + g) * kDD + 8 * i + 2 * c4) = make_float2(o[i][0], o[i][1]);
            *reinterpret_cast<float2*>(so + (warp * 16 + g + 8) * kDD + 8 * i + 2 * c4) = make_float2(o[i][2], o[i][3]);
        }
        if (c4 == 0) {
            *reinterpret_cast<float2*>(sml + (warp * 16 + g) * 2) = make_float2(m0, l0);
            *reinterpret_cast<float2*>(sml + (warp * 16 + g + 8) * 2) = make_float2(m1, l1);
        }
        __syncthreads();
        // thread t: row t / 8 (16 rows), 16 consecutive d values (t % 8)
        const int r = tid >> 3, d0 = (tid & 7) * 16;
        if (r < p.m_rows) {
            float mm = -INFINITY;
#pragma unroll
            for (int w = 0; w < 4; ++w) mm = fmaxf(mm, sml[(w * 16 + r) * 2]);
            float wt[4], L = 0.f;
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                const float mw = sml[(w * 16 + r) * 2];
                wt[w] = mw == -INFINITY ? 0.f : ex2f(mw - mm);
                L += wt[w] * sml[(w * 16 + r) * 2 + 1];
            }
            const int64_t base = (static_cast<int64_t>(h) * p.splits + split) * p.m_rows + r;
            float* dst = p.part_o + base * kDD + d0;
#pragma unroll
            for (int e = 0; e < 16; e += 4) {
                float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                    const float4 x = *reinterpret_cast<const float4*>(so + (w * 16 + r) * kDD + d0 + e);
                    acc.x += wt[w] * x.x;
                    acc.y += wt[w] * x.y;
                    acc.z += wt[w] * x.z;
                    acc.w += wt[w] * x.w;
                }
                *reinterpret_cast<float4*>(dst + e) = acc;
            }
            if ((tid & 7) == 0) *reinterpret_cast<float2*>(p.part_ml + base * 2) = make_float2(mm, L);
        }
        return;
    }
    const int qa = mtile * kQRows + warp * 16 + g, qb = qa + 8;
    const int64_t base = (static_cast<int64_t>(h) * p.splits + split) * p.m_rows;
    if (qa < p.m_rows) {
        float* dst = p.part_o + (base + qa) * kDD;
#pragma unroll
        for (int i = 0; i < kDD / 8; ++i) *reinterpret_cast<float2*>(dst + 8 * i + 2 * c4) = make_float2(o[i][0], o[i][1]);
        if (c4 == 0) *reinterpret_cast<float2*>(p.part_ml + (base + qa) * 2) = make_float2(m0, l0);
    }
    if (qb < p.m_rows) {
        float* dst = p.part_o + (base + qb) * kDD;
#pragma unroll
        for (int i = 0; i < kDD / 8; ++i) *reinterpret_cast<float2*>(dst + 8 * i + 2 * c4) = make_float2(o[i][2], o[i][3]);
        if (c4 == 0) *reinterpret_cast<float2*>(p.part_ml + (base + qb) * 2) = make_float2(m1, l1);
    }
}

// One CTA (8 warps) per (KV head, query row): merge the chunk partials (global max, rescaled sums), normalise, write
// O (bf16) and the natural-log LSE.  Warp w takes partials w, w + 8, ...; lane = 4 d values; smem tree at the end.
constexpr int kCombThreads = 256;
__global__ void __launch_bounds__(kCombThreads) decode_combine_kernel(const DecParams p, __nv_bfloat16* __restrict__ out,
                                                                      float* __restrict__ lse) {
    __shared__ float red[kCombThreads / 32][kDD + 1];
    __shared__ float smax[kCombThreads / 32];
    const int h = blockIdx.x / p.m_rows, qr = blockIdx.x - h * p.m_rows;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t row0 = static_cast<int64_t>(h) * p.splits * p.m_rows + qr;  // partial s at row0 + s * m_rows
    float mm = -INFINITY;
    for (int s = threadIdx.x; s < p.splits; s += kCombThreads)
        mm = fmaxf(mm, p.part_ml[(row0 + static_cast<int64_t>(s) * p.m_rows) * 2]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mm = fmaxf(mm, __shfl_xor_sync(0xffffffffu, mm, o));
    if (lane == 0) smax[warp] = mm;
    __syncthreads();
    mm = smax[0];
#pragma unroll
    for (int w = 1; w < kCombThreads / 32; ++w) mm = fmaxf(mm, smax[w]);
    float acc[4] = {0.f, 0.f, 0.f, 0.f}, L = 0.f;
    for (int s = warp; s < p.splits; s += kCombThreads / 32) {
        const int64_t idx = row0 + static_cast<int64_t>(s) * p.m_rows;
        const float2 ml = *reinterpret_cast<const float2*>(p.part_ml + idx * 2);
        const float w = ml.x == -INFINITY ? 0.f : ex2f(ml.x - mm);
        L += w * ml.y;
        const float4 v = *reinterpret_cast<const float4*>(p.part_o + idx * kDD + 4 * lane);
        acc[0] += w * v.x;
        acc[1] += w * v.y;
        acc[2] += w * v.z;
        acc[3] += w * v.w;
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) red[warp][4 * lane + e] = acc[e];
    if (lane == 0) red[warp][kDD] = L;
    __syncthreads();
    if (warp == 0) {
        float tot[4] = {0.f, 0.f, 0.f, 0.f}, LL = 0.f;
#pragma unroll
        for (int w = 0; w < kCombThreads / 32; ++w) {
#pragma unroll
            for (int e = 0; e < 4; ++e) tot[e] += red[w][4 * lane + e];
            LL += red[w][kDD];
        }
        const float inv = LL > 0.f ? 1.f / LL : 0.f;
        const int t = qr / p.group, hq = h * p.group + qr % p.group;
        __nv_bfloat16* dst = out + (static_cast<int64_t>(t) * p.n_q + hq) * kDD + 4 * lane;
        *reinterpret_cast<uint2*>(dst) =
            make_uint2(pack2(tot[0] * inv, tot[1] * inv), pack2(tot[2] * inv, tot[3] * inv));
        if (lse && lane == 0) lse[static_cast<int64_t>(t) * p.n_q + hq] = (mm + __log2f(LL)) * 0.6931471805599453f;
    }
}

// ---------------------------------------------------------------------------------------------------------------------
// tcgen05 variant for prompt-sized query batches (more than 16 query rows per KV head): the mma.sync kernel above is
// compute-bound there (~200 TFLOP/s).  A CTA takes two 128-row query tiles of one KV head and one chunk of cache
// rows, and runs the prefill kernel's ping-pong (attention.cu) without the causal mask: S_t = Q_t K(j)^T into TMEM,
// softmax in registers (thread = query row), P (bf16) written over S in TMEM, O_t += P V(j) with P as the TMEM
// operand; order PV0(j) S0(j+1) PV1(j) S1(j+1) so the tensor pipe works on one tile while the other's softmax runs.
// Q rows (token t, head h*g + i) are gathered by the softmax threads into the 128-byte-swizzled smem layout the UMMA
// descriptors expect; K / V blocks of 128 rows stream through a 4-stage TMA ring.  The chunk partials (unnormalised
// O, running max, sum) go to the same workspace as the mma.sync kernel's, merged by decode_combine_kernel.
constexpr int kTcThreads = 320;  // warps 0-3 softmax tile 0, 4-7 tile 1, 8 TMA, 9 MMA
constexpr int kTcStages = 4;
constexpr uint32_t kTcChunk = 128 * 128;      // one 128-row x 128-byte SW128 chunk (64 head-dim columns)
constexpr uint32_t kTcTile = 2 * kTcChunk;    // 128 rows x 128 d bf16
constexpr float kTcRescale = 8.0f;

struct TcBar {
    uint64_t q_ready;
    uint64_t kv_full[kTcStages], kv_empty[kTcStages];
    uint64_t s_full[2], p_full[2], o_done[2];
    uint32_t tmem_base;
};
constexpr size_t kTcSmem = 1024 + 2 * kTcTile + kTcStages * kTcTile + sizeof(TcBar);

__device__ __forceinline__ uint64_t tc_kdesc(uint32_t tile, int kk) {
    return ptx::umma_desc_sw128(tile + (kk >> 2) * kTcChunk + (kk & 3) * 32, 16, 1024);
}
__device__ __forceinline__ uint64_t tc_vdesc(uint32_t tile, int kk) {
    return ptx::umma_desc_sw128(tile + kk * 16 * 128, kTcChunk, 1024);
}

__global__ void __launch_bounds__(kTcThreads, 1)
    decode_tc_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                     const DecParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;                   // [tile][d chunk][128 rows x 128 B], swizzled
    uint8_t* sKV = smem + 2 * kTcTile;    // ring
    TcBar* bar = reinterpret_cast<TcBar*>(sKV + kTcStages * kTcTile);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int split = blockIdx.x, tp = blockIdx.y, h = blockIdx.z;
    const int64_t r_begin = static_cast<int64_t>(split) * p.rows_per_split;
    const int64_t r_end = min(p.rows, r_begin + p.rows_per_split);
    const int nb = static_cast<int>((r_end - r_begin + 127) / 128);
    const bool has1 = tp * 256 + 128 < p.m_rows;  // second query tile present

    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar->q_ready, 256);
        for (int s = 0; s < kTcStages; ++s) {
            ptx::mbar_init(&bar->kv_full[s], 1);
            ptx::mbar_init(&bar->kv_empty[s], 1);
        }
        for (int t = 0; t < 2; ++t) {
            ptx::mbar_init(&bar->s_full[t], 1);
            ptx::mbar_init(&bar->p_full[t], 128);
            ptx::mbar_init(&bar->o_done[t], 1);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 9) ptx::tmem_alloc<512>(&bar->tmem_base);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = bar->tmem_base;

    if (warp == 8) {
        if (ptx::elect_one()) {  // ===== TMA producer: K0 V0 K1 V1 ... =====
            ptx::prefetch_tmap(&tm_k);
            ptx::prefetch_tmap(&tm_v);
            for (int it = 0; it < 2 * nb; ++it) {
                const uint32_t st = it % kTcStages;
                ptx::mbar_wait(&bar->kv_empty[st], ((it / kTcStages) & 1) ^ 1);
                const CUtensorMap* map = (it & 1) ? &tm_v : &tm_k;
                const int row = static_cast<int>(r_begin) + (it >> 1) * 128;
                uint8_t* dst = sKV + st * kTcTile;
                ptx::mbar_arrive_expect_tx(&bar->kv_full[st], kTcTile);
                ptx::tma_load_3d(dst, map, &bar->kv_full[st], 0, h, row);
                ptx::tma_load_3d(dst + kTcChunk, map, &bar->kv_full[st], 64, h, row);
            }
        }
    } else if (warp == 9) {
        if (ptx::elect_one()) {  // ===== MMA issuer =====
            constexpr uint32_t kIdS = ptx::idesc_bf16_f32(128, 128, false, false);
            constexpr uint32_t kIdPV = ptx::idesc_bf16_f32(128, kDD, false, true);
            const uint32_t q_addr = ptx::smem_u32(sQ), ring = ptx::smem_u32(sKV);
            const int ntile = has1 ? 2 : 1;
            auto wait_item = [&](int it) -> uint32_t {
                const uint32_t st = it % kTcStages;
                ptx::mbar_wait(&bar->kv_full[st], (it / kTcStages) & 1);
                ptx::tc_fence_after();
                return ring + st * kTcTile;
            };
            auto issue_s = [&](int t, uint32_t k_addr) {
#pragma unroll
                for (int kk = 0; kk < kDD / 16; ++kk)
                    ptx::mma_ss(tmem + t * 128, tc_kdesc(q_addr + t * kTcTile, kk), tc_kdesc(k_addr, kk), kIdS, kk > 0);
                ptx::mma_commit(&bar->s_full[t]);
            };
            auto issue_pv = [&](int t, uint32_t v_addr, int j) {
                ptx::mbar_wait(&bar->p_full[t], j & 1);
                ptx::tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    ptx::mma_ts(tmem + 256 + t * 128, tmem + t * 128 + kk * 8, tc_vdesc(v_addr, kk), kIdPV,
                                (j > 0 || kk > 0) ? 1u : 0u);
                if (j == nb - 1) ptx::mma_commit(&bar->o_done[t]);
            };
            ptx::mbar_wait(&bar->q_ready, 0);
            ptx::tc_fence_after();
            const uint32_t k0 = wait_item(0);
            for (int t = 0; t < ntile; ++t) issue_s(t, k0);
            ptx::mma_commit(&bar->kv_empty[0]);
            for (int j = 0; j < nb; ++j) {
                const int v_it = 2 * j + 1;
                const uint32_t v_addr = wait_item(v_it);
                const bool more = j + 1 < nb;
                const uint32_t kn = more ? wait_item(v_it + 1) : 0u;
                issue_pv(0, v_addr, j);
                if (more) issue_s(0, kn);
                if (ntile > 1) {
                    issue_pv(1, v_addr, j);
                    if (more) issue_s(1, kn);
                }
                ptx::mma_commit(&bar->kv_empty[v_it % kTcStages]);
                if (more) ptx::mma_commit(&bar->kv_empty[(v_it + 1) % kTcStages]);
            }
        }
    } else {
        // ===== softmax (thread = query row of tile t) =====
        const int t = warp >> 2, quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
        const uint32_t s_col = tmem + lane_off + t * 128, o_col = tmem + lane_off + 256 + t * 128;
        const int qr = tp * 256 + t * 128 + row;  // query row of this KV head: token qr / g, head h*g + qr % g
        const bool live = qr < p.m_rows;
        {   // gather Q into the SW128 K-major layout (chunk c = d/64; 16-byte unit u of the 128-byte row at u ^ row%8)
            const int tok = live ? qr / p.group : 0, hq = h * p.group + (live ? qr % p.group : 0);
            const uint4* src = reinterpret_cast<const uint4*>(p.q + (static_cast<int64_t>(tok) * p.n_q + hq) * kDD);
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const uint4 x = live ? __ldg(src + u) : make_uint4(0u, 0u, 0u, 0u);
                const int c = u >> 3, uu = u & 7;
                ptx::sts128(ptx::smem_u32(sQ + t * kTcTile + c * kTcChunk + row * 128 + ((uu ^ (row & 7)) << 4)), x.x,
                            x.y, x.z, x.w);
            }
            ptx::fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the tensor cores
            ptx::mbar_arrive(&bar->q_ready);
        }
        const bool run = t == 0 || has1;
        const float sl2 = p.scale_log2;
        float m_ref = -INFINITY, l = 0.f;
        for (int j = 0; run && j < nb; ++j) {
            ptx::mbar_wait(&bar->s_full[t], j & 1);
            ptx::tc_fence_after();
            float x[128];
            QVK_TMEM_LD32F(s_col + 0, (x + 0));
            QVK_TMEM_LD32F(s_col + 32, (x + 32));
            QVK_TMEM_LD32F(s_col + 64, (x + 64));
            QVK_TMEM_LD32F(s_col + 96, (x + 96));
            ptx::tmem_ld_wait();
            const int64_t valid = r_end - (r_begin + static_cast<int64_t>(j) * 128);  // keys of this block in range
            if (valid < 128) {
#pragma unroll
                for (int c = 0; c < 128; ++c)
                    if (c >= valid) x[c] = -INFINITY;
            }
            float mx0 = x[0], mx1 = x[1], mx2 = x[2], mx3 = x[3];
#pragma unroll
            for (int c = 4; c < 128; c += 4) {
                mx0 = fmaxf(mx0, x[c]);
                mx1 = fmaxf(mx1, x[c + 1]);
                mx2 = fmaxf(mx2, x[c + 2]);
                mx3 = fmaxf(mx3, x[c + 3]);
            }
            const float m_new = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3)) * sl2;
            if (j == 0) {
                m_ref = m_new;
            } else {
                const bool need = m_new > m_ref + kTcRescale;
                if (__any_sync(0xffffffffu, need)) {  // the commit of S_t(j) proved PV_t(j-1) retired
                    const float m_upd = need ? m_new : m_ref;
                    const float f = ptx::ex2(m_ref - m_upd);
                    l *= f;
                    m_ref = m_upd;
#pragma unroll
                    for (int c = 0; c < kDD / 16; ++c) {
                        uint32_t o[16];
                        QVK_TMEM_LD16(o_col + c * 16, o);
                        ptx::tmem_ld_wait();
#pragma unroll
                        for (int e = 0; e < 16; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * f);
                        QVK_TMEM_ST16(o_col + c * 16, o);
                    }
                    ptx::tmem_st_wait();
                }
            }
            const ptx::f2 sl2x2 = ptx::f2_make(sl2, sl2), negx2 = ptx::f2_make(-m_ref, -m_ref);
            ptx::f2 acc0 = ptx::f2_make(0.f, 0.f), acc1 = acc0;
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                uint32_t pk[32];
#pragma unroll
                for (int c = 0; c < 32; ++c) {
                    const ptx::f2 y =
                        ptx::f2_fma(ptx::f2_make(x[64 * half + 2 * c], x[64 * half + 2 * c + 1]), sl2x2, negx2);
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
                QVK_TMEM_ST32(s_col + 32 * half, pk);
            }
            ptx::tmem_st_wait();
            ptx::tc_fence_before();
            ptx::mbar_arrive(&bar->p_full[t]);
            float s0, s1, s2, s3;
            ptx::f2_split(acc0, s0, s1);
            ptx::f2_split(acc1, s2, s3);
            l += (s0 + s1) + (s2 + s3);
        }
        if (run) {
            ptx::mbar_wait(&bar->o_done[t], 0);
            ptx::tc_fence_after();
            const int64_t base = (static_cast<int64_t>(h) * p.splits + split) * p.m_rows + qr;
#pragma unroll
            for (int c = 0; c < kDD / 16; ++c) {
                uint32_t o[16];
                QVK_TMEM_LD16(o_col + c * 16, o);
                ptx::tmem_ld_wait();
                if (live) {
                    float4* dst = reinterpret_cast<float4*>(p.part_o + base * kDD + c * 16);
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        dst[e] = make_float4(__uint_as_float(o[4 * e]), __uint_as_float(o[4 * e + 1]),
                                             __uint_as_float(o[4 * e + 2]), __uint_as_float(o[4 * e + 3]));
                }
            }
            if (live) *reinterpret_cast<float2*>(p.part_ml + base * 2) = make_float2(m_ref, l);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 9) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tmem);
    }
}

bool dec_map(CUtensorMap* m, const void* base, int heads, int64_t rows) {
    const auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(tensor_map_encoder());
    if (!enc) return false;
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(kDD), static_cast<cuuint64_t>(heads), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(kDD) * 2, static_cast<cuuint64_t>(heads) * kDD * 2};
    cuuint32_t box[3] = {64, 1, 128};
    cuuint32_t estr[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

int launch_decode_attention(cudaStream_t stream, const void* q, int n_tq, int n_q, int n_kv, int d_h,
                            const void* k_cache, const void* v_cache, int64_t rows, float scale, void* o, float* lse,
                            void* ws, size_t ws_bytes, size_t* ws_needed) {
    if (d_h != kDD) {
        set_error("decode_attention: head_dim must be 128");
        return QVK_E_UNSUPPORTED;
    }
    if (n_tq <= 0 || n_q <= 0 || n_kv <= 0 || n_q % n_kv != 0)
        QVK_INVALID("decode_attention: n_q must be a positive multiple of n_kv");
    if (rows <= 0) QVK_INVALID("decode_attention: empty cache");
    if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k_cache) | reinterpret_cast<uintptr_t>(v_cache) |
         reinterpret_cast<uintptr_t>(o)) & 15)
        QVK_INVALID("decode_attention: tensors must be 16-byte aligned");
    DecParams p;
    p.q = static_cast<const __nv_bfloat16*>(q);
    p.k = static_cast<const __nv_bfloat16*>(k_cache);
    p.v = static_cast<const __nv_bfloat16*>(v_cache);
    p.rows = rows;
    p.n_tq = n_tq;
    p.n_q = n_q;
    p.n_kv = n_kv;
    p.group = n_q / n_kv;
    p.m_rows = n_tq * p.group;
    p.scale_log2 = scale * 1.4426950408889634f;
    static const int tc_env = env_knob("QVK_DECODE_TC", 1) != 0;  // 0: prompt batches on the mma.sync kernel
    const bool tc = tc_env && p.m_rows > 16 && rows <= 0x7fffffff;
    const int mtiles = tc ? (p.m_rows + 255) / 256 : (p.m_rows + kQRows - 1) / kQRows;  // tc: pairs of 128-row tiles
    const int rows_blk = tc ? 128 : kKvRows;
    const int64_t blocks = (rows + rows_blk - 1) / rows_blk;
    const int64_t base = static_cast<int64_t>(mtiles) * n_kv;
    const bool ws_mode = !tc && p.m_rows <= 16;
    const int64_t per_sm = tc ? 2 : 4;  // target CTAs per SM worth of chunks
    int64_t splits = std::max<int64_t>(1, std::min<int64_t>(blocks, (per_sm * kNumSms + base - 1) / base));
    const int64_t blocks_per = (blocks + splits - 1) / splits;
    splits = (blocks + blocks_per - 1) / blocks_per;
    if (blocks_per * rows_blk > 0x7fffffff || splits > 16383 || mtiles > 65535)
        QVK_INVALID("decode_attention: problem too large");
    p.rows_per_split = static_cast<int>(blocks_per * rows_blk);
    p.splits = static_cast<int>(splits);  // partials per (KV head, query row): one per chunk
    const size_t part = static_cast<size_t>(n_kv) * p.splits * p.m_rows;
    const size_t need = part * kDD * sizeof(float) + part * 2 * sizeof(float);
    if (ws_needed) *ws_needed = need;
    if (!ws) {
        if (ws_needed) return QVK_OK;  // size query
        QVK_INVALID("decode_attention: workspace required");
    }
    if (ws_bytes < need) QVK_INVALID("decode_attention: workspace too small");
    p.part_o = static_cast<float*>(ws);
    p.part_ml = p.part_o + part * kDD;
    const dim3 grid(tc ? static_cast<unsigned>(splits) : static_cast<unsigned>(mtiles),
                    tc ? static_cast<unsigned>(mtiles) : static_cast<unsigned>(splits), n_kv);
    if (tc) {
        CUtensorMap mk, mv;
        if (!dec_map(&mk, k_cache, n_kv, rows) || !dec_map(&mv, v_cache, n_kv, rows)) {
            set_error("decode_attention: cuTensorMapEncodeTiled failed");
            return QVK_E_CUDA;
        }
        QVK_CUDA_CHECK(func_attr(reinterpret_cast<const void*>(decode_tc_kernel),
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kTcSmem)));
        decode_tc_kernel<<<grid, kTcThreads, kTcSmem, stream>>>(mk, mv, p);
    } else {
        constexpr size_t smem = (kQRows + 4 * kKvRows) * kPad * sizeof(__nv_bfloat16);
        QVK_CUDA_CHECK(func_attr(reinterpret_cast<const void*>(decode_attention_kernel<true>),
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        QVK_CUDA_CHECK(func_attr(reinterpret_cast<const void*>(decode_attention_kernel<false>),
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        if (ws_mode)
            decode_attention_kernel<true><<<grid, kDecThreads, smem, stream>>>(p);
        else
            decode_attention_kernel<false><<<grid, kDecThreads, smem, stream>>>(p);
    }
    QVK_LAUNCH_CHECK();
    decode_combine_kernel<<<static_cast<unsigned>(n_kv * p.m_rows), kCombThreads, 0, stream>>>(
        p, static_cast<__nv_bfloat16*>(o), lse);
    QVK_LAUNCH_CHECK();
    return QVK_OK;
}

}  // namespace qvk
