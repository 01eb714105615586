/* Plain C99 caller of the C ABI (include/qvk.h only — no CUDA headers, no C++): plan the groups of a small
 * video, upload per-KV-head bf16 keys / values, prune every group in one qvk_prune call (score -> top-k ->
 * compaction, prefill.cpp:255-282 batched) and read the cache back.  This is the binding surface a caller in
 * another language (cgo, JNI, ctypes, N-API) sees.
 *
 *   gcc -std=c99 -O2 -Iinclude examples/c_abi_prune.c -Lpaper_2505_16175_b200/lib -lqvk \
 *       -Wl,-rpath,$PWD/paper_2505_16175_b200/lib -o c_abi_prune && ./c_abi_prune [out.bin]
 *
 * Inputs are a deterministic LCG (same as tests/test_c_abi_gpu.py); with an output path the retained indices
 * (uint32, (cache row, head)) and the K cache (bf16 bits) are written there for the test to compare. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "qvk.h"

#define CHECK(call)                                                                       \
    do {                                                                                  \
        int rc_ = (call);                                                                 \
        if (rc_ != QVK_OK) {                                                              \
            fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, qvk_last_error());       \
            return 1;                                                                     \
        }                                                                                 \
    } while (0)

static uint16_t to_bf16(float f) { /* round to nearest even */
    uint32_t u;
    memcpy(&u, &f, 4);
    return (uint16_t)((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
}

int main(int argc, char** argv) {
    const uint64_t frames = 16;
    const uint32_t fpg = 4, tpf = 64;
    const int32_t heads = 2, width = 128;
    const double rho = 0.5;
    uint64_t G = 0;
    CHECK(qvk_plan_groups(frames, fpg, tpf, rho, 1, &G, NULL, NULL, NULL, NULL));
    int64_t* tok_off = malloc(sizeof(int64_t) * (G + 1));
    int64_t* keep = malloc(sizeof(int64_t) * G);
    int64_t* row_off = malloc(sizeof(int64_t) * (G + 1));
    uint64_t* first = malloc(sizeof(uint64_t) * G);
    CHECK(qvk_plan_groups(frames, fpg, tpf, rho, 1, &G, tok_off, keep, row_off, NULL));
    for (uint64_t g = 0; g < G; ++g) first[g] = (uint64_t)tok_off[g];
    const int64_t T = tok_off[G], R = row_off[G];
    const size_t n = (size_t)T * heads * width;
    uint16_t* k = malloc(n * 2);
    uint16_t* v = malloc(n * 2);
    uint64_t s = 0x9e3779b97f4a7c15ull;
    for (size_t i = 0; i < n; ++i) { /* LCG -> uniform [-1, 1) */
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        k[i] = to_bf16((float)((double)(s >> 11) / 9007199254740992.0 * 2.0 - 1.0));
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        v[i] = to_bf16((float)((double)(s >> 11) / 9007199254740992.0 * 2.0 - 1.0));
    }
    void *k_d, *v_d, *kc_d, *vc_d, *tok_d, *keep_d, *row_d, *first_d, *idx_d, *org_d;
    CHECK(qvk_malloc(&k_d, n * 2));
    CHECK(qvk_malloc(&v_d, n * 2));
    CHECK(qvk_malloc(&kc_d, (size_t)R * heads * width * 2));
    CHECK(qvk_malloc(&vc_d, (size_t)R * heads * width * 2));
    CHECK(qvk_malloc(&idx_d, (size_t)R * heads * 4));
    CHECK(qvk_malloc(&org_d, (size_t)R * heads * 8));
    CHECK(qvk_malloc(&tok_d, sizeof(int64_t) * (G + 1)));
    CHECK(qvk_malloc(&keep_d, sizeof(int64_t) * G));
    CHECK(qvk_malloc(&row_d, sizeof(int64_t) * (G + 1)));
    CHECK(qvk_malloc(&first_d, sizeof(uint64_t) * G));
    CHECK(qvk_memcpy_h2d(k_d, k, n * 2, NULL));
    CHECK(qvk_memcpy_h2d(v_d, v, n * 2, NULL));
    CHECK(qvk_memcpy_h2d(tok_d, tok_off, sizeof(int64_t) * (G + 1), NULL));
    CHECK(qvk_memcpy_h2d(keep_d, keep, sizeof(int64_t) * G, NULL));
    CHECK(qvk_memcpy_h2d(row_d, row_off, sizeof(int64_t) * (G + 1), NULL));
    CHECK(qvk_memcpy_h2d(first_d, first, sizeof(uint64_t) * G, NULL));
    int64_t max_n = 0;
    for (uint64_t g = 0; g < G; ++g)
        if (tok_off[g + 1] - tok_off[g] > max_n) max_n = tok_off[g + 1] - tok_off[g];
    qvk_groups groups = {(int32_t)G, max_n, T, R, tok_d, keep_d, row_d, first_d};
    CHECK(qvk_prune(NULL, &groups, k_d, v_d, QVK_BF16, heads, width, QVK_KEY_NORM_SMALL, rho, NULL, 0, heads, NULL,
                    idx_d, kc_d, vc_d, org_d));
    uint32_t* idx = malloc((size_t)R * heads * 4);
    uint16_t* kc = malloc((size_t)R * heads * width * 2);
    uint64_t* org = malloc((size_t)R * heads * 8);
    CHECK(qvk_memcpy_d2h(idx, idx_d, (size_t)R * heads * 4, NULL));
    CHECK(qvk_memcpy_d2h(kc, kc_d, (size_t)R * heads * width * 2, NULL));
    CHECK(qvk_memcpy_d2h(org, org_d, (size_t)R * heads * 8, NULL));
    CHECK(qvk_stream_sync(NULL));
    /* structural checks: per (group, head) ascending indices, origins, copied rows */
    for (uint64_t g = 0; g < G; ++g)
        for (int32_t h = 0; h < heads; ++h)
            for (int64_t r = 0; r < keep[g]; ++r) {
                const int64_t cr = (row_off[g] + r) * heads + h;
                const uint32_t j = idx[cr];
                if ((r > 0 && idx[cr - heads] >= j) || org[cr] != first[g] + j ||
                    memcmp(kc + cr * width, k + ((tok_off[g] + j) * heads + h) * width, width * 2) != 0) {
                    fprintf(stderr, "mismatch at group %llu head %d row %lld\n", (unsigned long long)g, h,
                            (long long)r);
                    return 1;
                }
            }
    if (argc > 1) {
        FILE* f = fopen(argv[1], "wb");
        if (!f) return 1;
        fwrite(idx, 4, (size_t)R * heads, f);
        fwrite(kc, 2, (size_t)R * heads * width, f);
        fclose(f);
    }
    printf("c_abi_prune ok: %llu groups, %lld tokens, %lld cache rows x %d heads\n", (unsigned long long)G,
           (long long)T, (long long)R, heads);
    void* bufs[] = {k_d, v_d, kc_d, vc_d, idx_d, org_d, tok_d, keep_d, row_d, first_d};
    for (int i = 0; i < 10; ++i) CHECK(qvk_free(bufs[i]));
    return 0;
}
