// Developer microbenchmark (not part of the product): single-warp-per-SMSP throughput of the softmax instruction mix.
#include <cstdio>
#include <cstdint>
#include "../paper_2505_16175_b200/csrc/ptx.cuh"

template <int kMode, int kWarps>
__global__ void bench(const float* in, uint32_t* out, long long* cyc, int iters) {
    float x[64];
    for (int i = 0; i < 64; ++i) x[i] = in[(threadIdx.x + i) & 255] - 3.f;
    uint32_t acc = 0;
    float facc = 0.f;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        uint32_t pk[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) {
            float p0, p1;
            if (kMode == 0) {  // MUFU only
                p0 = qvk::ptx::ex2(x[2 * c]);
                p1 = qvk::ptx::ex2(x[2 * c + 1]);
                pk[c] = __float_as_uint(p0) ^ __float_as_uint(p1);
            } else if (kMode == 1) {  // MUFU + F2FP
                p0 = qvk::ptx::ex2(x[2 * c]);
                p1 = qvk::ptx::ex2(x[2 * c + 1]);
                pk[c] = qvk::ptx::pack_bf16(p0, p1);
            } else if (kMode == 2) {  // F2FP only
                pk[c] = qvk::ptx::pack_bf16(x[2 * c], x[2 * c + 1]);
            } else if (kMode == 3) {  // poly only
                p0 = x[2 * c]; p1 = x[2 * c + 1];
                qvk::ptx::ex2_poly2(p0, p1);
                pk[c] = __float_as_uint(p0) ^ __float_as_uint(p1);
            } else if (kMode == 5) {  // bf16x2 ex2: pack, one MUFU per pair
                uint32_t in2 = qvk::ptx::pack_bf16(x[2 * c], x[2 * c + 1]);
                uint32_t o2;
                asm("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(o2) : "r"(in2));
                pk[c] = o2;
            } else if (kMode == 6) {  // full bf16 path: FFMA2 scale, pack, ex2.bf16x2, unpack + FADD2 sum
                const qvk::ptx::f2 y = qvk::ptx::f2_fma(qvk::ptx::f2_make(x[2 * c], x[2 * c + 1]),
                                                        qvk::ptx::f2_make(1.01f, 1.01f),
                                                        qvk::ptx::f2_make(-0.5f, -0.5f));
                qvk::ptx::f2_split(y, p0, p1);
                uint32_t in2 = qvk::ptx::pack_bf16(p0, p1);
                uint32_t o2;
                asm("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(o2) : "r"(in2));
                facc += __uint_as_float(o2 << 16) + __uint_as_float(o2 & 0xffff0000u);
                pk[c] = o2;
            } else if (kMode == 7) {  // scalar FFMA chain poly (no packed ops)
                p0 = x[2 * c]; p1 = x[2 * c + 1];
                #pragma unroll
                for (int e = 0; e < 2; ++e) {
                    float& z = e ? p1 : p0;
                    const float cz = fmaxf(z, -126.f);
                    const float t = cz + 12582912.f;
                    const float fr = cz - (t - 12582912.f);
                    float q = fmaf(fr, 0.05517146f, 0.24261086f);
                    q = fmaf(q, fr, 0.69326097f);
                    q = fmaf(q, fr, 0.9999281f);
                    z = __uint_as_float(__float_as_uint(q) + (__float_as_uint(t) << 23));
                }
                pk[c] = __float_as_uint(p0) ^ __float_as_uint(p1);
            } else {  // full mix as in the kernel (FFMA2 scale, MUFU, FADD2 sum, F2FP)
                const qvk::ptx::f2 y = qvk::ptx::f2_fma(qvk::ptx::f2_make(x[2 * c], x[2 * c + 1]),
                                                        qvk::ptx::f2_make(1.01f, 1.01f),
                                                        qvk::ptx::f2_make(-0.5f, -0.5f));
                qvk::ptx::f2_split(y, p0, p1);
                p0 = qvk::ptx::ex2(p0);
                p1 = qvk::ptx::ex2(p1);
                facc += p0 + p1;
                pk[c] = qvk::ptx::pack_bf16(p0, p1);
            }
        }
#pragma unroll
        for (int c = 0; c < 32; ++c) acc += pk[c];
#pragma unroll
        for (int i = 0; i < 64; ++i) x[i] = __uint_as_float(__float_as_uint(x[i]) ^ (acc & 1));
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc + __float_as_uint(facc);
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int kMode, int kWarps>
void run(const char* name, const float* in, uint32_t* out, long long* cyc) {
    const int iters = 1000;
    bench<kMode, kWarps><<<148, 32 * kWarps>>>(in, out, cyc, iters);
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    // per warp: iters * 64 elements
    printf("%-14s warps/CTA %2d: %.2f cycles per 64-element block per warp, %.2f cycles/element/SMSP\n", name, kWarps,
           double(c) / iters, double(c) / iters / 64 / (kWarps / 4.0 > 1 ? kWarps / 4.0 : 1));
}

int main() {
    float* in; uint32_t* out; long long* cyc;
    cudaMalloc(&in, 256 * 4); cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
    cudaMemset(in, 0, 1024);
    run<0, 4>("mufu", in, out, cyc); run<0, 8>("mufu", in, out, cyc); run<0, 16>("mufu", in, out, cyc);
    run<1, 4>("mufu+f2fp", in, out, cyc); run<1, 8>("mufu+f2fp", in, out, cyc);
    run<2, 4>("f2fp", in, out, cyc); run<2, 8>("f2fp", in, out, cyc);
    run<3, 4>("poly", in, out, cyc); run<3, 8>("poly", in, out, cyc);
    run<5, 4>("ex2bf16x2", in, out, cyc); run<5, 8>("ex2bf16x2", in, out, cyc); run<5, 16>("ex2bf16x2", in, out, cyc);
    run<6, 4>("full-bf16", in, out, cyc); run<6, 8>("full-bf16", in, out, cyc); run<6, 16>("full-bf16", in, out, cyc);
    run<7, 4>("poly-scalar", in, out, cyc); run<7, 8>("poly-scalar", in, out, cyc); run<7, 16>("poly-scalar", in, out, cyc);
    run<4, 4>("full", in, out, cyc); run<4, 8>("full", in, out, cyc); run<4, 16>("full", in, out, cyc);
    return 0;
}
