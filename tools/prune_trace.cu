// Developer tool (not part of the product): per-CTA phase timeline of the fused prune kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DQVK_PRUNE_TRACE -Iinclude \
//        -Ipaper_2505_16175_b200/csrc tools/prune_trace.cu -o build/prune_trace && build/prune_trace [G N heads]
// Builds prune_fused.cu with QVK_PRUNE_TRACE, runs key-norm pruning at rho 0.5 on G groups x N tokens x heads x 128
// (default: the C2 shape 16 x 4096 x 4) after an L2 flush and prints, per phase boundary, the min / median / max
// over CTAs of the %globaltimer offset from the earliest CTA start (ns).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "../paper_2505_16175_b200/csrc/prune_fused.cu"

namespace qvk {
void set_error(const std::string& m) { fprintf(stderr, "qvk error: %s\n", m.c_str()); }
int env_knob(const char* name, int def) {
    const char* e = getenv(name);
    return e ? atoi(e) : def;
}
cudaError_t func_attr(const void* f, cudaFuncAttribute a, int v) { return cudaFuncSetAttribute(f, a, v); }
}

__global__ void fill(__nv_bfloat16* p, size_t n, uint32_t seed) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint32_t h = (uint32_t)i * 2654435761u ^ seed;
        h ^= h >> 15; h *= 0x2c1b3c6du; h ^= h >> 12;
        p[i] = __float2bfloat16(((h & 0xffff) / 65535.f - 0.5f) * 3.f);
    }
}

int main(int argc, char** argv) {
    const int G = argc > 1 ? atoi(argv[1]) : 16, N = argc > 2 ? atoi(argv[2]) : 4096;
    const int H = argc > 3 ? atoi(argv[3]) : 4, D = 128;
    const int64_t T = (int64_t)G * N, keep = N / 2, R = (int64_t)G * keep;
    __nv_bfloat16 *k, *v, *kc, *vc;
    cudaMalloc(&k, T * H * D * 2); cudaMalloc(&v, T * H * D * 2);
    cudaMalloc(&kc, R * H * D * 2); cudaMalloc(&vc, R * H * D * 2);
    double* sc; cudaMalloc(&sc, T * H * 8);
    uint32_t* idx; cudaMalloc(&idx, R * H * 4);
    uint64_t* org; cudaMalloc(&org, R * H * 8);
    fill<<<1024, 256>>>(k, T * H * D, 2); fill<<<1024, 256>>>(v, T * H * D, 3);
    std::vector<int64_t> off(G + 1), kp(G), ro(G + 1);
    std::vector<uint64_t> ft(G);
    for (int g = 0; g <= G; ++g) { off[g] = (int64_t)g * N; ro[g] = (int64_t)g * keep; }
    for (int g = 0; g < G; ++g) { kp[g] = keep; ft[g] = off[g]; }
    int64_t *off_d, *kp_d, *ro_d; uint64_t* ft_d;
    cudaMalloc(&off_d, 8 * (G + 1)); cudaMalloc(&kp_d, 8 * G); cudaMalloc(&ro_d, 8 * (G + 1)); cudaMalloc(&ft_d, 8 * G);
    cudaMemcpy(off_d, off.data(), 8 * (G + 1), cudaMemcpyHostToDevice);
    cudaMemcpy(kp_d, kp.data(), 8 * G, cudaMemcpyHostToDevice);
    cudaMemcpy(ro_d, ro.data(), 8 * (G + 1), cudaMemcpyHostToDevice);
    cudaMemcpy(ft_d, ft.data(), 8 * G, cudaMemcpyHostToDevice);
    qvk_groups grp{G, N, T, R, off_d, kp_d, ro_d, ft_d};
    const int ctas = G * H * 16;
    uint32_t* tr; cudaMalloc(&tr, ctas * 8 * 4);
    cudaMemcpyToSymbol(qvk::g_prune_trace, &tr, sizeof(tr));
    uint32_t* smid; cudaMalloc(&smid, ctas * 4);
    cudaMemcpyToSymbol(qvk::g_prune_smid, &smid, sizeof(smid));
    void* flush; cudaMalloc(&flush, 256 << 20);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms = 0;
    for (int it = 0; it < 4; ++it) {
        cudaMemset(tr, 0, ctas * 8 * 4);
        cudaMemsetAsync(flush, it, 256 << 20);
        cudaEventRecord(e0);
        int rc = qvk::launch_prune_fused(0, &grp, k, v, H, D, QVK_KEY_NORM_SMALL, nullptr, sc, idx, kc, vc, org, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (rc) { printf("rc %d\n", rc); return 1; }
    }
    std::vector<uint32_t> h(ctas * 8);
    cudaMemcpy(h.data(), tr, h.size() * 4, cudaMemcpyDeviceToHost);
    int used = 0;
    uint32_t t0 = 0xffffffffu;
    for (int c = 0; c < ctas; ++c) if (h[c * 8]) { ++used; t0 = std::min(t0, h[c * 8]); }
    printf("G=%d N=%d heads=%d: %.1f us (event), %d CTAs traced\n", G, N, H, ms * 1e3, used);
    const char* names[8] = {"start", "scored", "lo/hi agreed", "selected", "compacted", "gathered", "scores out", "exit"};
    for (int s = 0; s < 8; ++s) {
        std::vector<uint32_t> x;
        for (int c = 0; c < used; ++c) x.push_back(h[c * 8 + s] - t0);
        std::sort(x.begin(), x.end());
        printf("%-14s min %7u  p50 %7u  p90 %7u  max %7u ns\n", names[s], x[0], x[x.size() / 2], x[x.size() * 9 / 10],
               x.back());
    }
    // SM load: CTAs per SM, and the scoring time (start -> scored) of CTAs by the load of their SM
    std::vector<uint32_t> sm(ctas);
    cudaMemcpy(sm.data(), smid, ctas * 4, cudaMemcpyDeviceToHost);
    std::vector<int> load(256, 0);
    std::vector<int> rounds(32, 0);
    for (int c = 0; c < used; ++c) ++rounds[std::min(31u, sm[c] >> 16)];
    printf("select rounds per CTA:");
    for (int r = 0; r < 32; ++r)
        if (rounds[r]) printf("  %d: %d", r, rounds[r]);
    printf("\n");
    for (auto& x : sm) x &= 0xffffu;
    for (int c = 0; c < used; ++c) ++load[sm[c]];
    int sms = 0;
    for (int i = 0; i < 256; ++i) sms += load[i] > 0;
    printf("SMs used %d\n", sms);
    for (int l = 1; l <= 16; ++l) {
        std::vector<uint32_t> x, y;
        for (int c = 0; c < used; ++c)
            if (load[sm[c]] == l) { x.push_back(h[c * 8 + 1] - h[c * 8]); y.push_back(h[c * 8 + 1] - t0); }
        if (x.empty()) continue;
        std::sort(x.begin(), x.end());
        std::sort(y.begin(), y.end());
        printf("SM load %2d: %4zu CTAs  score dur p50 %6u max %6u | scored at p50 %6u max %6u ns\n", l, x.size(),
               x[x.size() / 2], x.back(), y[y.size() / 2], y.back());
    }
    return 0;
}
