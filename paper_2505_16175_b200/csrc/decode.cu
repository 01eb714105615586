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
#include "common.cuh"

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
    const int mtiles = (p.m_rows + kQRows - 1) / kQRows;
    const int64_t blocks = (rows + kKvRows - 1) / kKvRows;
    const int64_t base = static_cast<int64_t>(mtiles) * n_kv;
    const bool ws_mode = p.m_rows <= 16;
    int64_t splits = std::max<int64_t>(1, std::min<int64_t>(blocks, (4 * kNumSms + base - 1) / base));
    const int64_t blocks_per = (blocks + splits - 1) / splits;
    splits = (blocks + blocks_per - 1) / blocks_per;
    if (blocks_per * kKvRows > 0x7fffffff || splits > 16383 || mtiles > 65535)
        QVK_INVALID("decode_attention: problem too large");
    p.rows_per_split = static_cast<int>(blocks_per * kKvRows);
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
    constexpr size_t smem = (kQRows + 4 * kKvRows) * kPad * sizeof(__nv_bfloat16);
    QVK_CUDA_CHECK(func_attr(reinterpret_cast<const void*>(decode_attention_kernel<true>),
                             cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    QVK_CUDA_CHECK(func_attr(reinterpret_cast<const void*>(decode_attention_kernel<false>),
                             cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    const dim3 grid(mtiles, static_cast<unsigned>(splits), n_kv);
    if (ws_mode)
        decode_attention_kernel<true><<<grid, kDecThreads, smem, stream>>>(p);
    else
        decode_attention_kernel<false><<<grid, kDecThreads, smem, stream>>>(p);
    QVK_LAUNCH_CHECK();
    decode_combine_kernel<<<static_cast<unsigned>(n_kv * p.m_rows), kCombThreads, 0, stream>>>(
        p, static_cast<__nv_bfloat16*>(o), lse);
    QVK_LAUNCH_CHECK();
    return QVK_OK;
}

}  // namespace qvk
