// Developer microbenchmark (not part of the product): B200 throughput of F2F.F64.F32, DFMA, integer-built doubles.
#include <cstdio>
#include <cstdint>

template <int kMode>
__global__ void bench(const uint32_t* in, double* out, long long* cyc, int iters) {
    uint32_t w[8];
    for (int i = 0; i < 8; ++i) w[i] = in[(threadIdx.x + i) & 255] | 0x3f803f80u;
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const uint32_t bits = q ? (w[i] & 0xffff0000u) : (w[i] << 16);
                double d;
                if (kMode == 0) {  // F2F
                    d = static_cast<double>(__uint_as_float(bits));
                } else {  // integer-built |x| (normal bf16 only)
                    const uint32_t a = bits >> 16 & 0x7fffu;
                    const uint32_t hi = a ? (a << 13) + 0x38000000u : 0u;
                    d = __hiloint2double(static_cast<int>(hi), 0);
                }
                if (kMode == 2) d = static_cast<double>(__uint_as_float(bits));  // F2F only, no DFMA chain below
                if ((i * 2 + q) % 4 == 0) acc0 = __fma_rn(d, d, acc0);
                else if ((i * 2 + q) % 4 == 1) acc1 = __fma_rn(d, d, acc1);
                else if ((i * 2 + q) % 4 == 2) acc2 = __fma_rn(d, d, acc2);
                else acc3 = __fma_rn(d, d, acc3);
            }
            w[i] = w[i] * 1664525u + 1013904223u;
        }
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1 + acc2 + acc3;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int kMode>
void run(const char* name, int threads, const uint32_t* in, double* out, long long* cyc) {
    const int iters = 2000;
    bench<kMode><<<148, threads>>>(in, out, cyc, iters);
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double elems = double(iters) * 16 * threads;  // per SM
    printf("%-12s threads %4d: %.2f elements/clk/SM\n", name, threads, elems / c);
}

int main() {
    uint32_t* in; double* out; long long* cyc;
    cudaMalloc(&in, 1024); cudaMalloc(&out, 148 * 1024 * 8); cudaMalloc(&cyc, 148 * 8);
    cudaMemset(in, 0x11, 1024);
    for (int t : {128, 256, 512, 1024}) {
        run<0>("f2f+dfma", t, in, out, cyc);
        run<1>("int+dfma", t, in, out, cyc);
    }
    return 0;
}
