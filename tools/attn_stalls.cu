// Developer tool (not part of the product): where the attention kernel's MMA issuer waits.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DQVK_ATTN_STALLS -Iinclude \
//        -Ipaper_2505_16175_b200/csrc tools/attn_stalls.cu -lcuda -o build/attn_stalls && build/attn_stalls [G N]
// Builds attention.cu with QVK_ATTN_STALLS and prints, averaged over CTAs, the cycles per unit the MMA warp spent
// waiting on each barrier (Q loaded, K/V tile loaded, O released by the epilogue, P published by the softmax), the
// tile-0 softmax's wait for S, and the epilogue's wait for l / O.
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
    void* sym; cudaGetSymbolAddress(&sym, qvk::g_attn_stall);
    cudaMemset(sym, 0, sizeof(unsigned long long) * 1024 * 8);
    cudaEventRecord(e0);
    int rc = qvk::launch_attention(0, &grp, q, k, v, nq, nkv, d, 0.0883883f, o);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (rc) { printf("rc %d\n", rc); return 1; }
    std::vector<unsigned long long> h(1024 * 8);
    cudaMemcpy(h.data(), sym, h.size() * 8, cudaMemcpyDeviceToHost);
    double tot[8] = {0};
    int ctas = 0;
    for (int c = 0; c < 1024; ++c) {
        if (!h[c * 8 + 5]) continue;
        ++ctas;
        for (int k2 = 0; k2 < 8; ++k2) tot[k2] += h[c * 8 + k2];
    }
    const double units = tot[5];
    const double flops = 4.0 * d * nq * (double)N * (N + 1) / 2 * G;
    printf("G=%d N=%d: %.3f ms  %.0f TFLOP/s  %d CTAs  %.1f units/CTA  MMA loop %.0f cycles/CTA -> %.0f MHz\n", G, N,
           ms, flops / ms / 1e9, ctas, units / ctas, tot[4] / ctas, tot[4] / ctas / (ms * 1e3));
    const char* names[8] = {"MMA q_full", "MMA kv_full", "MMA o_free", "MMA p_full", "MMA loop", "units",
                            "softmax0 s_full", "epilogue l/o"};
    for (int k2 = 0; k2 < 8; ++k2)
        if (k2 != 5) printf("  %-16s %9.0f cycles per unit  (%.1f %% of the MMA loop)\n", names[k2], tot[k2] / units,
                            100.0 * tot[k2] / tot[4]);
    return 0;
}
