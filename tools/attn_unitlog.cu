// Developer tool (not part of the product): per-unit cost of the attention kernel over EVERY CTA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DQVK_ATTN_UNITLOG -Iinclude \
//        -Ipaper_2505_16175_b200/csrc tools/attn_unitlog.cu -lcuda -o build/attn_unitlog && build/attn_unitlog 16 4096
// The MMA thread stamps clock64 at the top of each unit; unit i's cost = stamp(i+1) - stamp(i) (the time the MMA
// thread spends from one unit's start to the next's, i.e. the unit's steady-state pace including its boundary).
// Prints the mean cost per K/V-step count and the least-squares fit cost = a * nkv + b (a = cycles per K/V step of
// two tiles, b = per-unit overhead).
#include <cstdio>
#include <cstdlib>
#include <map>
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
    const int G = argc > 1 ? atoi(argv[1]) : 16, N = argc > 2 ? atoi(argv[2]) : 4096, nq = 28, nkv = 4, d = 128;
    const int64_t T = (int64_t)G * N;
    __nv_bfloat16 *q, *k, *v, *o;
    cudaMalloc(&q, T * nq * d * 2);
    cudaMalloc(&o, T * nq * d * 2);
    cudaMalloc(&k, T * nkv * d * 2);
    cudaMalloc(&v, T * nkv * d * 2);
    fill<<<1024, 256>>>(q, T * nq * d, 1);
    fill<<<1024, 256>>>(k, T * nkv * d, 2);
    fill<<<1024, 256>>>(v, T * nkv * d, 3);
    std::vector<int64_t> off(G + 1);
    for (int g = 0; g <= G; ++g) off[g] = (int64_t)g * N;
    int64_t* off_d;
    cudaMalloc(&off_d, 8 * (G + 1));
    cudaMemcpy(off_d, off.data(), 8 * (G + 1), cudaMemcpyHostToDevice);
    qvk_groups grp{G, N, T, T / 2, off_d, off_d, off_d, nullptr};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int it = 0; it < 3; ++it) qvk::launch_attention(0, &grp, q, k, v, nq, nkv, d, 0.0883883f, o);
    static long long zero[1024][129][3];
    cudaMemcpyToSymbol(qvk::g_attn_unitlog, zero, sizeof(zero));
    cudaEventRecord(e0);
    int rc = qvk::launch_attention(0, &grp, q, k, v, nq, nkv, d, 0.0883883f, o);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double tf = G * 4.0 * d * nq * (double)N * (N + 1) / 2 / (ms * 1e-3) / 1e12;
    static long long lg[1024][129][3];
    cudaMemcpyFromSymbol(lg, qvk::g_attn_unitlog, sizeof(lg));
    int sms = qvk::sm_count();
    std::map<long long, std::pair<double, long long>> by;  // nkv -> (sum cycles, count)
    double sx = 0, sy = 0, sxx = 0, sxy = 0, n = 0, tot = 0, first = 1e30, last = 0, cyc = 0, ns = 0;
    long long steps = 0;
    for (int c = 0; c < sms; ++c) {
        int i = 0;
        for (; i < 128 && lg[c][i + 1][0]; ++i) {
            const double dur = double(lg[c][i + 1][0] - lg[c][i][0]);
            const long long x = lg[c][i][1];
            by[x].first += dur;
            by[x].second += 1;
            sx += x;
            sy += dur;
            sxx += double(x) * x;
            sxy += x * dur;
            n += 1;
            steps += x;
        }
        if (i > 0) {
            tot += double(lg[c][i][0] - lg[c][0][0]);
            cyc += double(lg[c][i][0] - lg[c][0][0]);
            ns += double(lg[c][i][2] - lg[c][0][2]);
            first = std::min(first, double(lg[c][0][0]));
            last = std::max(last, double(lg[c][i][0]));
        }
    }
    const double a = (n * sxy - sx * sy) / (n * sxx - sx * sx), b = (sy - a * sx) / n;
    printf("G=%d N=%d rc=%d err=%s  %.3f ms  %.1f TFLOP/s  units logged %.0f  mean CTA loop %.0f cycles\n", G, N, rc,
           cudaGetErrorString(err), ms, tf, n, tot / sms);
    printf("SM clock over the logged spans: %.0f MHz\n", ns > 0 ? cyc / ns * 1e3 : 0.0);
    printf("fit: cycles per unit = %.1f * nkv + %.1f   (mean K/V steps per unit %.2f)\n", a, b, sx / n);
    printf(" nkv  units  mean cycles  cycles/step\n");
    for (auto& kv : by)
        printf("%4lld %6lld %12.0f %12.1f\n", kv.first, kv.second.second, kv.second.first / kv.second.second,
               kv.second.first / kv.second.second / kv.first);
    return 0;
}
