// Stand-in model pieces of the reference API, computed on the device and bit-identical to prefill.cpp:
//   seeded_matrix   prefill.cpp:21-30   counter-based splitmix64, double arithmetic, float store
//   project_exact   prefill.cpp:38-54   out = x * w with double accumulation in the reference's sequential order
//   tokenize        prefill.cpp:123-168 per-patch double mean (exact integer sums) and the 3 -> d embed
// plus the synthetic bf16 generator of the benchmark (same bits as oracle qvo_synth_bf16).
// Every double operation is an explicit _rn intrinsic, so nvcc never contracts a rounding the reference performs into
// an FMA; the projection's FMAs are exact by construction (see project_exact_kernel).
#include "common.cuh"

namespace qvk {
namespace {

__global__ void seeded_matrix_kernel(uint64_t state0, size_t count, double scale, float* __restrict__ out) {
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const double u = __dmul_rn(static_cast<double>(splitmix64_at(state0, i) >> 11), 0x1.0p-53);
        out[i] = __double2float_rn(__dmul_rn(__dsub_rn(__dmul_rn(u, 2.0), 1.0), scale));
    }
}

// out(rows, d_out) = x(rows, d_in) * w(d_in, d_out): every output accumulates i = 0..d_in-1 in order, in double
// (prefill.cpp:38-54 `acc[o] += xi * wrow[o]`).  The product of two floats is exact in double (24 + 24 bits), so
// fma(xi, w, acc) rounds exactly like acc + xi * w: bit-identical to the reference while running one DFMA per MAC.
// CTA tile 64 rows x 64 outputs, 256 threads with 4 x 4 outputs each (register tile), reduction chunks of 32
// staged in shared memory as doubles (converted once per element, not per use).  Shared-memory layout chosen for
// the banks (the first version was bound by bank conflicts: ncu L1 94 %, FP64 pipe 23 %): the x tile's rows are
// padded to 66 doubles, so the transposing stores hit distinct bank pairs; a thread's
// four outputs are columns {2 tx, 2 tx + 1, 32 + 2 tx, 33 + 2 tx}, so each 16-byte w load of a warp covers 256
// contiguous bytes (two wavefronts, no conflict).
constexpr int kPM = 64, kPN = 64, kPK = 32, kPXS = kPM + 2;
__global__ void __launch_bounds__(256) project_exact_kernel(const float* __restrict__ x, int64_t rows, int d_in,
                                                            const float* __restrict__ w, int d_out,
                                                            float* __restrict__ out) {
    __shared__ __align__(16) double xs[kPK][kPXS];  // xs[i][r]
    __shared__ __align__(16) double ws[kPK][kPN];   // ws[i][o]
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // outputs {2tx, 2tx+1, 32+2tx, 33+2tx}, rows 4ty..
    const int64_t r0 = static_cast<int64_t>(blockIdx.y) * kPM;
    const int o0 = blockIdx.x * kPN;
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    for (int i0 = 0; i0 < d_in; i0 += kPK) {
        __syncthreads();
        // x tile: a warp covers 2 rows x 16 consecutive i (64-byte row segments); with the 66-double rows its 32
        // transposing stores land on distinct bank pairs two by two (the minimum two wavefronts)
        for (int e = threadIdx.x; e < kPM * kPK; e += 256) {
            const int e2 = e % (kPM * 16);
            const int rr = e2 / 16, ii = (e / (kPM * 16)) * 16 + (e2 % 16);
            const int64_t gr = r0 + rr;
            xs[ii][rr] = (gr < rows && i0 + ii < d_in) ? static_cast<double>(__ldg(x + gr * d_in + i0 + ii)) : 0.0;
        }
        for (int e = threadIdx.x; e < kPK * kPN; e += 256) {
            const int ii = e / kPN, oo = e % kPN;
            const int go = o0 + oo;
            ws[ii][oo] = (go < d_out && i0 + ii < d_in)
                             ? static_cast<double>(__ldg(w + static_cast<int64_t>(i0 + ii) * d_out + go)) : 0.0;
        }
        __syncthreads();
        const int kw = min(kPK, d_in - i0);
#pragma unroll 4
        for (int ii = 0; ii < kw; ++ii) {
            const double2 xa = *reinterpret_cast<const double2*>(&xs[ii][ty * 4]);
            const double2 xb = *reinterpret_cast<const double2*>(&xs[ii][ty * 4 + 2]);
            const double2 wa = *reinterpret_cast<const double2*>(&ws[ii][2 * tx]);
            const double2 wb = *reinterpret_cast<const double2*>(&ws[ii][32 + 2 * tx]);
            const double xv[4] = {xa.x, xa.y, xb.x, xb.y}, wv[4] = {wa.x, wa.y, wb.x, wb.y};
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b] = __fma_rn(xv[a], wv[b], acc[a][b]);
        }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int64_t r = r0 + ty * 4 + a;
        if (r >= rows) continue;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int o = o0 + (b < 2 ? 2 * tx + b : 32 + 2 * tx + (b - 2));
            if (o < d_out) out[r * d_out + o] = __double2float_rn(acc[a][b]);
        }
    }
}

// One CTA per token (frame slot f, patch gr, gc).  Integer channel sums are exact in any order (the reference
// accumulates uint8 into a double, exact below 2^53), then mean = sum / (double(ph) * pw) and
// out[o] = float(e0*m0 + e1*m1 + e2*m2) evaluated left to right in double.
// OutT float: the reference's fp32 tokens bit for bit; __nv_bfloat16: the same fp32 value rounded to bf16 (RNE), the
// activations of the bf16 projection GEMM (frames -> pruned cache path, pipeline.py FramePrefill).
template <typename OutT>
__global__ void __launch_bounds__(256) tokenize_kernel(const uint8_t* __restrict__ frames, uint32_t width,
                                                       uint32_t height, uint32_t tpf, uint32_t grid_cols,
                                                       uint32_t ph, uint32_t pw, const float* __restrict__ embed,
                                                       int d, OutT* __restrict__ tokens) {
    __shared__ unsigned long long sums[3];
    __shared__ double mean[3];
    const int64_t token = blockIdx.x;
    const int64_t f = token / tpf;
    const uint32_t p = static_cast<uint32_t>(token - f * tpf);
    const uint32_t gr = p / grid_cols, gc = p % grid_cols;
    const size_t plane = static_cast<size_t>(width) * height;
    const uint8_t* px = frames + f * 3 * plane;
    if (threadIdx.x < 3) sums[threadIdx.x] = 0;
    __syncthreads();
    unsigned long long part[3] = {0, 0, 0};
    for (uint32_t e = threadIdx.x; e < ph * pw; e += blockDim.x) {
        const uint32_t y = gr * ph + e / pw, x = gc * pw + e % pw;
#pragma unroll
        for (int c = 0; c < 3; ++c) part[c] += px[c * plane + static_cast<size_t>(y) * width + x];
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) atomicAdd(&sums[c], part[c]);
    __syncthreads();
    if (threadIdx.x < 3)
        mean[threadIdx.x] = __ddiv_rn(static_cast<double>(sums[threadIdx.x]),
                                      __dmul_rn(static_cast<double>(ph), static_cast<double>(pw)));
    __syncthreads();
    for (int o = threadIdx.x; o < d; o += blockDim.x) {
        const double e0 = embed[o * 3 + 0], e1 = embed[o * 3 + 1], e2 = embed[o * 3 + 2];
        const double s = __dadd_rn(__dadd_rn(__dmul_rn(e0, mean[0]), __dmul_rn(e1, mean[1])), __dmul_rn(e2, mean[2]));
        const float f = __double2float_rn(s);
        if constexpr (sizeof(OutT) == 4) tokens[token * d + o] = f;
        else tokens[token * d + o] = __float2bfloat16_rn(f);
    }
}

// Throughput variant of the same tokenizer (identical values): a CTA takes kTokCta consecutive tokens (patches) of one
// frame.  Patch sums: 4 threads per patch, 4 bytes per load (__dp4a), exact integer sums reduced by shuffles, then
// the reference's double mean.  Embed: each thread owns the outputs o = tid (mod 256) and converts their 3 embed
// weights to double ONCE for all kTokCta tokens (the per-token kernel above reconverts them for every token), then
// writes o for every token of the CTA (coalesced across the warp).
constexpr int kTokCta = 64;
template <typename OutT>
__global__ void __launch_bounds__(256) tokenize_fast_kernel(const uint8_t* __restrict__ frames, uint32_t width,
                                                            uint32_t height, uint32_t tpf, uint32_t grid_cols,
                                                            uint32_t ph, uint32_t pw, const float* __restrict__ embed,
                                                            int d, OutT* __restrict__ tokens) {
    __shared__ double mean[kTokCta][3];
    const int64_t f = blockIdx.x;
    const uint32_t p0 = blockIdx.y * kTokCta;
    const uint32_t np = min(static_cast<uint32_t>(kTokCta), tpf - p0);
    const size_t plane = static_cast<size_t>(width) * height;
    const uint8_t* px = frames + f * 3 * plane;
    {
        const uint32_t pl = threadIdx.x >> 2, part = threadIdx.x & 3;
        uint32_t acc[3] = {0u, 0u, 0u};
        if (pl < np) {
            const uint32_t p = p0 + pl, gr = p / grid_cols, gc = p % grid_cols;
            // 32-bit loads need every row start 4-byte aligned: pw, width and the frames pointer itself
            const bool vec = (pw % 4 == 0) && (width % 4 == 0) && (reinterpret_cast<uintptr_t>(frames) & 3) == 0;
            for (uint32_t y = part; y < ph; y += 4) {
                const size_t row = static_cast<size_t>(gr * ph + y) * width + gc * pw;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const uint8_t* r = px + c * plane + row;
                    if (vec) {
                        for (uint32_t x = 0; x < pw; x += 4)
                            acc[c] = __dp4a(*reinterpret_cast<const uint32_t*>(r + x), 0x01010101u, acc[c]);
                    } else {
                        for (uint32_t x = 0; x < pw; ++x) acc[c] += r[x];
                    }
                }
            }
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], 1);
            acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], 2);
        }
        if (pl < np && part == 0) {
            const double cnt = __dmul_rn(static_cast<double>(ph), static_cast<double>(pw));
#pragma unroll
            for (int c = 0; c < 3; ++c) mean[pl][c] = __ddiv_rn(static_cast<double>(acc[c]), cnt);
        }
    }
    __syncthreads();
    OutT* out = tokens + (f * tpf + p0) * static_cast<int64_t>(d);
    for (int o = threadIdx.x; o < d; o += blockDim.x) {
        const double e0 = embed[o * 3 + 0], e1 = embed[o * 3 + 1], e2 = embed[o * 3 + 2];
        for (uint32_t t = 0; t < np; ++t) {
            const double s =
                __dadd_rn(__dadd_rn(__dmul_rn(e0, mean[t][0]), __dmul_rn(e1, mean[t][1])), __dmul_rn(e2, mean[t][2]));
            const float v = __double2float_rn(s);
            if constexpr (sizeof(OutT) == 4) out[t * static_cast<int64_t>(d) + o] = v;
            else out[t * static_cast<int64_t>(d) + o] = __float2bfloat16_rn(v);
        }
    }
}

__constant__ float kHeadScale[9] = {0.5f,        0.59460356f, 0.70710678f, 0.84089642f, 1.0f,
                                    1.18920712f, 1.41421356f, 1.68179283f, 2.0f};

// Irwin-Hall(4) approximate N(0,1) per element, per-(row, head) scale 2^(j/4); see oracle qvo_synth_bf16.
__global__ void synth_bf16_kernel(uint64_t base, int64_t rows, int heads, int width, int head_scale,
                                  __nv_bfloat16* __restrict__ out) {
    const int64_t total = rows * heads * width;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint64_t z = splitmix64_at(base, static_cast<uint64_t>(e));
        const int32_t s = static_cast<int32_t>(z & 0xffff) + static_cast<int32_t>((z >> 16) & 0xffff) +
                          static_cast<int32_t>((z >> 32) & 0xffff) + static_cast<int32_t>(z >> 48);
        float val = __fmul_rn(static_cast<float>(s - 131070), 2.6428812e-05f);
        if (head_scale) {
            const uint64_t unit = static_cast<uint64_t>(e / width);
            val = __fmul_rn(val, kHeadScale[splitmix64_at(base ^ 0x5bd1e995ull, unit) % 9]);
        }
        out[e] = __float2bfloat16_rn(val);
    }
}

unsigned grid_for(int64_t n, int threads) {
    const int64_t want = (n + threads - 1) / threads;
    return static_cast<unsigned>(want < 1 ? 1 : (want > kNumSms * 32 ? kNumSms * 32 : want));
}

}  // namespace

int launch_seeded_matrix(cudaStream_t s, uint64_t seed, uint32_t tag, uint32_t layer, size_t count, double scale,
                         float* out) {
    if (count == 0) return QVK_OK;
    seeded_matrix_kernel<<<grid_for(static_cast<int64_t>(count), 256), 256, 0, s>>>(stream_seed(seed, tag, layer),
                                                                                    count, scale, out);
    QVK_LAUNCH_CHECK();
    return QVK_OK;
}

int launch_project_exact(cudaStream_t s, const float* x, int64_t rows, int d_in, const float* w, int d_out,
                         float* out) {
    if (rows == 0 || d_out == 0) return QVK_OK;
    if ((rows + kPM - 1) / kPM > 65535) QVK_INVALID("project: too many rows for one launch");
    dim3 grid((d_out + kPN - 1) / kPN, static_cast<unsigned>((rows + kPM - 1) / kPM));
    project_exact_kernel<<<grid, 256, 0, s>>>(x, rows, d_in, w, d_out, out);
    QVK_LAUNCH_CHECK();
    return QVK_OK;
}

int launch_tokenize(cudaStream_t s, const uint8_t* frames, int64_t n_frames, uint32_t width, uint32_t height,
                    uint32_t tpf, uint32_t grid_rows, uint32_t grid_cols, const float* embed, int d, void* tokens,
                    int bf16_out) {
    const int64_t n_tok = n_frames * tpf;
    if (n_tok == 0) return QVK_OK;
    if (n_tok > 0x7fffffff) QVK_INVALID("tokenize: too many tokens for one launch");
    const uint32_t ph = height / grid_rows, pw = width / grid_cols;
    if (n_frames <= 0x7fffffff && ph * pw <= (1u << 24)) {  // u32 patch sums: at most 2^24 pixels of <= 255
        const dim3 grid(static_cast<unsigned>(n_frames), (tpf + kTokCta - 1) / kTokCta);
        if (bf16_out)
            tokenize_fast_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(frames, width, height, tpf, grid_cols, ph, pw,
                                                                     embed, d, static_cast<__nv_bfloat16*>(tokens));
        else
            tokenize_fast_kernel<float><<<grid, 256, 0, s>>>(frames, width, height, tpf, grid_cols, ph, pw, embed, d,
                                                             static_cast<float*>(tokens));
    } else if (bf16_out) {
        tokenize_kernel<__nv_bfloat16><<<static_cast<unsigned>(n_tok), 256, 0, s>>>(
            frames, width, height, tpf, grid_cols, ph, pw, embed, d, static_cast<__nv_bfloat16*>(tokens));
    } else {
        tokenize_kernel<float><<<static_cast<unsigned>(n_tok), 256, 0, s>>>(
            frames, width, height, tpf, grid_cols, ph, pw, embed, d, static_cast<float*>(tokens));
    }
    QVK_LAUNCH_CHECK();
    return QVK_OK;
}

int launch_synth_bf16(cudaStream_t s, uint64_t seed, uint32_t tag, uint32_t layer, uint64_t group, int64_t rows,
                      int heads, int width, int head_scale, void* out) {
    const uint64_t base = stream_seed(seed, tag, layer) ^ (group * 0xd1b54a32d192ed03ull);
    const int64_t total = rows * heads * width;
    if (total == 0) return QVK_OK;
    synth_bf16_kernel<<<grid_for(total, 256), 256, 0, s>>>(base, rows, heads, width, head_scale,
                                                           static_cast<__nv_bfloat16*>(out));
    QVK_LAUNCH_CHECK();
    return QVK_OK;
}

}  // namespace qvk
