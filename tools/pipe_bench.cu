// Developer microbenchmark (not part of the product): per-SMSP reciprocal throughput of the instructions the
// attention softmax is built from (FFMA, FFMA2, FADD2, MUFU.EX2, F2FP.BF16 pack, FMNMX, FMNMX3, IMAD, HFMA2.BF16),
// 8 independent dependency chains per thread, 1 / 2 / 4 warps per SM sub-partition.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_bench tools/pipe_bench.cu && ./pipe_bench
#include <cstdint>
#include <cstdio>

#include "../paper_2505_16175_b200/csrc/ptx.cuh"

using qvk::ptx::f2;

template <int kOp>
__device__ __forceinline__ void step(float (&a)[16], uint32_t (&u)[16]) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        if (kOp == 0) {  // FFMA (3 registers)
            a[i] = fmaf(a[i], a[i + 8], a[(i + 1) & 7]);
        } else if (kOp == 1) {  // FFMA2
            f2 x = qvk::ptx::f2_make(a[2 * (i & 3)], a[2 * (i & 3) + 1]);
            f2 y = qvk::ptx::f2_make(a[8 + 2 * (i & 3)], a[9 + 2 * (i & 3)]);
            f2 r = qvk::ptx::f2_fma(x, y, x);
            qvk::ptx::f2_split(r, a[2 * (i & 3)], a[2 * (i & 3) + 1]);
        } else if (kOp == 2) {  // FADD2
            f2 x = qvk::ptx::f2_make(a[2 * (i & 3)], a[2 * (i & 3) + 1]);
            f2 y = qvk::ptx::f2_make(a[8 + 2 * (i & 3)], a[9 + 2 * (i & 3)]);
            f2 r = qvk::ptx::f2_add(x, y);
            qvk::ptx::f2_split(r, a[2 * (i & 3)], a[2 * (i & 3) + 1]);
        } else if (kOp == 3) {  // MUFU.EX2
            a[i] = qvk::ptx::ex2(a[i]);
        } else if (kOp == 4) {  // F2FP pack
            u[i] = qvk::ptx::pack_bf16(a[i] + __uint_as_float(u[i]), a[i + 8]);
        } else if (kOp == 5) {  // FMNMX
            a[i] = fmaxf(a[i], a[i + 8]);
        } else if (kOp == 6) {  // FMNMX3
            float d;
            asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a[i]), "f"(a[i + 8]), "f"(a[(i + 9) & 15]));
            a[i] = d;
        } else if (kOp == 7) {  // IMAD
            u[i] = u[i] * u[i + 8] + u[(i + 1) & 7];
        } else if (kOp == 8) {  // HFMA2.BF16 (packed bf16 fma)
            uint32_t d;
            asm volatile("fma.rn.bf16x2 %0, %1, %2, %3;" : "=r"(d) : "r"(u[i]), "r"(u[i + 8]), "r"(u[(i + 1) & 7]));
            u[i] = d;
        } else if (kOp == 9) {  // FADD (2 registers)
            a[i] = a[i] + a[i + 8];
        } else if (kOp == 10) {  // FFMA with immediates
            a[i] = fmaf(a[i], 1.0001f, 0.5f);
        } else if (kOp == 11) {  // FMUL2 via fma.rn.f32x2 with zero addend replaced by mul
            f2 x = qvk::ptx::f2_make(a[2 * (i & 3)], a[2 * (i & 3) + 1]);
            f2 y = qvk::ptx::f2_make(a[8 + 2 * (i & 3)], a[9 + 2 * (i & 3)]);
            f2 r;
            asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(x.v), "l"(y.v));
            qvk::ptx::f2_split(r, a[2 * (i & 3)], a[2 * (i & 3) + 1]);
        }
    }
}

template <int kOp>
__global__ void bench(const float* in, uint32_t* out, long long* cyc, int iters) {
    float a[16];
    uint32_t u[16];
    for (int i = 0; i < 16; ++i) {
        a[i] = in[(threadIdx.x + i) & 255];
        u[i] = __float_as_uint(a[i]);
    }
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        step<kOp>(a, u);
        step<kOp>(a, u);
        step<kOp>(a, u);
        step<kOp>(a, u);
    }
    const long long t1 = clock64();
    uint32_t acc = 0;
    for (int i = 0; i < 16; ++i) acc += __float_as_uint(a[i]) + u[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int kOp>
void run(const char* name, const float* in, uint32_t* out, long long* cyc) {
    const int iters = 2000;
    for (int wps = 1; wps <= 4; wps *= 2) {
        bench<kOp><<<148, 128 * wps>>>(in, out, cyc, iters);
        cudaDeviceSynchronize();
        long long c;
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        // instructions per warp: iters * 4 steps * 8
        const double per = double(c) / (double(iters) * 32) / wps;
        printf("%-10s warps/SMSP %d: %.2f cycles per warp-instruction per SMSP\n", name, wps, per);
    }
}

int main() {
    float* in;
    uint32_t* out;
    long long* cyc;
    cudaMalloc(&in, 256 * 4);
    cudaMalloc(&out, 148 * 1024 * 4);
    cudaMalloc(&cyc, 148 * 8);
    float h[256];
    for (int i = 0; i < 256; ++i) h[i] = 0.25f + 0.001f * i;
    cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
    run<0>("FFMA", in, out, cyc);
    run<10>("FFMA-imm", in, out, cyc);
    run<9>("FADD", in, out, cyc);
    run<1>("FFMA2", in, out, cyc);
    run<2>("FADD2", in, out, cyc);
    run<11>("FMUL2", in, out, cyc);
    run<3>("MUFU.EX2", in, out, cyc);
    run<4>("F2FP+FADD", in, out, cyc);
    run<5>("FMNMX", in, out, cyc);
    run<6>("FMNMX3", in, out, cyc);
    run<7>("IMAD", in, out, cyc);
    run<8>("HFMA2.BF16", in, out, cyc);
    return 0;
}
