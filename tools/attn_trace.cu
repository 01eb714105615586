// Developer tool (not part of the product): timeline of one attention CTA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DQVK_ATTN_TRACE -Iinclude \
//        -Ipaper_2505_16175_b200/csrc tools/attn_trace.cu -lcuda -o build/attn_trace && build/attn_trace
// Builds attention.cu with QVK_ATTN_TRACE, runs the C2 shape (16 groups x 4096 tokens, 28/4 heads, d 128) and prints
// the clock64 stamps CTA 0 (the heaviest query-tile pair of group 0, head 0) recorded per K/V step.  Add
// -DQVK_ATTN_TRACE_UNITS=4 (and run e.g. `64 1024`) to trace CTA 0's first four units, rows 8u..8u+7; the `prolog`
// column of rows 8u..8u+4 holds unit u's prologue stamps (S1(0) issued, K(0) ready, decoded, Q ready, loop top) and
// row 8u+nkv-1 the time its last MMA was issued.
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "../paper_2505_16175_b200/csrc/attention.cu"

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
int launch_attention2(cudaStream_t, const qvk_groups*, const void*, const void*, const void*, int, int, float, void*) {
    return QVK_E_UNSUPPORTED;
}
}

__global__ void fill(__nv_bfloat16* p, size_t n, uint32_t seed) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint32_t h = (uint32_t)i * 2654435761u ^ seed;
        h ^= h >> 15; h *= 0x2c1b3c6du; h ^= h >> 12;
        p[i] = __float2bfloat16(((h & 0xffff) / 65535.f - 0.5f) * 3.f);
    }
}

int main(int argc, char** argv) {
    const int G = argc > 1 ? atoi(argv[1]) : 16, N = argc > 2 ? atoi(argv[2]) : 4096, nq = 28, nkv = 4, d = 128;
    const int64_t T = (int64_t)G * N;
    __nv_bfloat16 *q, *k, *v, *o;
    cudaMalloc(&q, T * nq * d * 2); cudaMalloc(&o, T * nq * d * 2);
    cudaMalloc(&k, T * nkv * d * 2); cudaMalloc(&v, T * nkv * d * 2);
    fill<<<1024, 256>>>(q, T * nq * d, 1); fill<<<1024, 256>>>(k, T * nkv * d, 2); fill<<<1024, 256>>>(v, T * nkv * d, 3);
    std::vector<int64_t> off(G + 1);
    for (int g = 0; g <= G; ++g) off[g] = (int64_t)g * N;
    int64_t* off_d; cudaMalloc(&off_d, 8 * (G + 1));
    cudaMemcpy(off_d, off.data(), 8 * (G + 1), cudaMemcpyHostToDevice);
    qvk_groups grp{G, N, T, T / 2, off_d, off_d, off_d, nullptr};
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int it = 0; it < 3; ++it) qvk::launch_attention(0, &grp, q, k, v, nq, nkv, d, 0.0883883f, o);
    cudaEventRecord(e0);
    int rc = qvk::launch_attention(0, &grp, q, k, v, nq, nkv, d, 0.0883883f, o);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("rc=%d err=%s  %.3f ms  %.1f TFLOP/s\n", rc, cudaGetErrorString(err), ms,
           G * 4.0 * d * nq * (double)N * (N + 1) / 2 / (ms * 1e-3) / 1e12);
#ifndef QVK_ATTN_TRACE
    return 0;
#else
    long long tr[1024];
    cudaMemcpyFromSymbol(tr, qvk::g_attn_trace, sizeof(tr));
    const long long t0 = tr[1022];
    printf("  j |  V rdy   P0h0   P0h1  S0iss   P1h0   P1h1  S1iss  prolog || sm0:S rdy  max   h0    h1 | sm1:S rdy  max   h0    h1\n");
    for (int j = 0; j < 32; ++j) {
        printf("%3d |", j);
        for (int e = 0; e < 8; ++e) printf(" %6lld", tr[j * 8 + e] ? (tr[j * 8 + e] - t0) : -1);
        printf(" ||");
        for (int t = 0; t < 2; ++t) {
            for (int e = 0; e < 4; ++e) {
                long long x = tr[512 + t * 256 + j * 8 + e];
                printf(" %6lld", x ? x - t0 : -1);
            }
            printf(" |");
        }
        printf("\n");
    }
    printf("o_done seen: tile0 %lld tile1 %lld\n", tr[512 + 255] - t0, tr[768 + 255] - t0);
    return 0;
#endif
}
