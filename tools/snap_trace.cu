// Developer tool (not part of the product): per-key-tile timeline of the SnapKV tcgen05 kernel (CTA 0, its first
// two items) and the launch time.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DQVK_SNAP_TRACE -Iinclude \
//        -Ipaper_2505_16175_b200/csrc tools/snap_trace.cu -lcuda -o build/tools/snap_trace && build/tools/snap_trace 64 1024
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "../paper_2505_16175_b200/csrc/snapkv.cu"

namespace qvk {
void set_error(const std::string& m) { fprintf(stderr, "qvk error: %s\n", m.c_str()); }
int sm_count() {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, 0);
    return v;
}
void* tensor_map_encoder() {
    cudaDriverEntryPointQueryResult q;
    void* ptr = nullptr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q);
    return ptr;
}
int env_knob(const char* name, int def) {
    const char* e = getenv(name);
    return e ? atoi(e) : def;
}
cudaError_t func_attr(const void* f, cudaFuncAttribute a, int v) { return cudaFuncSetAttribute(f, a, v); }
cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t s) { return cudaMallocAsync(p, bytes, s); }
}  // namespace qvk

__global__ void fill(__nv_bfloat16* p, size_t n, uint32_t seed) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint32_t h = (uint32_t)i * 2654435761u ^ seed;
        h ^= h >> 15;
        h *= 0x2c1b3c6du;
        h ^= h >> 12;
        p[i] = __float2bfloat16(((h & 0xffff) / 65535.f - 0.5f) * 3.f);
    }
}

int main(int argc, char** argv) {
    const int G = argc > 1 ? atoi(argv[1]) : 64, N = argc > 2 ? atoi(argv[2]) : 1024, nq = 28, nkv = 4, d = 128;
    const int64_t T = (int64_t)G * N;
    __nv_bfloat16 *q, *k;
    double* sc;
    cudaMalloc(&q, T * nq * d * 2);
    cudaMalloc(&k, T * nkv * d * 2);
    cudaMalloc(&sc, T * nkv * 8);
    fill<<<1024, 256>>>(q, T * nq * d, 1);
    fill<<<1024, 256>>>(k, T * nkv * d, 2);
    std::vector<int64_t> off(G + 1);
    for (int g = 0; g <= G; ++g) off[g] = (int64_t)g * N;
    int64_t* off_d;
    cudaMalloc(&off_d, 8 * (G + 1));
    cudaMemcpy(off_d, off.data(), 8 * (G + 1), cudaMemcpyHostToDevice);
    qvk_groups grp{G, N, T, T / 4, off_d, off_d, off_d, nullptr};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    // argv[3] == "p2": pass 2 alone on (arbitrary, finite) window statistics, as the layer path runs it
    const bool p2 = argc > 3 && std::string(argv[3]) == "p2";
    float* lse = nullptr;
    if (p2) {
        cudaMalloc(&lse, sizeof(float) * G * nq * 32);
        cudaMemset(lse, 0, sizeof(float) * G * nq * 32);
    }
    for (int it = 0; it < 3; ++it) qvk::launch_snapkv(0, &grp, q, k, nq, nkv, d, 32, 1, 0.0883883f, sc, lse, 0);
    static long long zero[2][64][10];
    cudaMemcpyToSymbol(qvk::g_snap_trace, zero, sizeof(zero));
    float best = 1e9;
    for (int it = 0; it < 5; ++it) {
        unsigned long long span0[3] = {~0ull, 0ull, 0ull};
        cudaMemcpyToSymbol(qvk::g_snap_span, span0, sizeof(span0));
        cudaEventRecord(e0);
        qvk::launch_snapkv(0, &grp, q, k, nq, nkv, d, 32, 1, 0.0883883f, sc, lse, 0);
        cudaEventRecord(e1);
        cudaDeviceSynchronize();
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms);
    }
    printf("G=%d N=%d %s err=%s  best of 5: %.1f us\n", G, N, p2 ? "pass 2 alone" : "two passes",
           cudaGetErrorString(cudaGetLastError()), best * 1e3);
    {
        unsigned long long span[3];
        cudaMemcpyFromSymbol(span, qvk::g_snap_span, sizeof(span));
        printf("last launch: CTAs from first start to last end %.1f us\n", (span[1] - span[0]) * 1e-3);
    }
    static long long tr[2][64][10];
    cudaMemcpyFromSymbol(tr, qvk::g_snap_trace, sizeof(tr));
    const long long t0 = tr[0][0][0];
    const int nt = (N + 127) / 128;
    {  // effective SM clock over CTA 0's traced span: clock64 cycles / globaltimer ns
        long long c0 = tr[0][0][0], g0 = tr[0][0][9], c1 = 0, g1 = 0;
        for (int it = 0; it < 2; ++it)
            for (int t = 0; t < 64; ++t)
                if (tr[it][t][0] && tr[it][t][9]) c1 = tr[it][t][0], g1 = tr[it][t][9];
        if (g1 > g0) printf("SM clock over the traced span: %.0f MHz\n", double(c1 - c0) / double(g1 - g0) * 1e3);
    }
    printf("item tile | MMA: wait  issue  done || w0: full  rel  math || w13: full  rel  math   (cycles from item 0 tile 0)\n");
    for (int it = 0; it < 2; ++it)
        for (int t = 0; t < 2 * nt && t < 64; ++t) {
            printf("%4d %4d |", it, t);
            for (int s = 0; s < 9; ++s) {
                printf(" %7lld", tr[it][t][s] ? tr[it][t][s] - t0 : -1);
                if (s == 2 || s == 5) printf(" ||");
            }
            printf("\n");
        }
    return 0;
}
