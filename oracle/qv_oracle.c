/* TEST INFRASTRUCTURE ONLY — CPU restatement of the QuickPrefill hot path (see qv_oracle.h for the contract).
 * Built with -ffp-contract=off (oracle/Makefile) so no double expression is contracted into an FMA. */
#include "qv_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

uint64_t qvo_splitmix64(uint64_t* state) { /* synthetic.cpp:5-10 */
    uint64_t z = (*state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

uint64_t qvo_stream_seed(uint64_t seed, uint32_t tag, uint32_t layer) { /* prefill.cpp:13-18 */
    uint64_t s = seed;
    s = s * 0x100000001b3ull + tag + 1;
    s = s * 0x100000001b3ull + layer + 1;
    return s;
}

void qvo_seeded_matrix(uint64_t seed, uint32_t tag, uint32_t layer, size_t count, double scale, float* out) {
    /* prefill.cpp:21-30 */
    uint64_t state = qvo_stream_seed(seed, tag, layer);
    for (size_t i = 0; i < count; ++i) {
        const double u = (double)(qvo_splitmix64(&state) >> 11) * 0x1.0p-53;
        out[i] = (float)((u * 2.0 - 1.0) * scale);
    }
}

float qvo_bf16_to_f32(uint16_t b) {
    uint32_t u = (uint32_t)b << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

uint16_t qvo_f32_to_bf16(float f) { /* round to nearest even; NaN kept quiet */
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40);
    u += 0x7fffu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

/* 2^(j/4), j = -4..4, as exact float literals (shared with csrc/synth.cu). */
static const float kHeadScale[9] = {0.5f,       0.59460356f, 0.70710678f, 0.84089642f, 1.0f,
                                    1.18920712f, 1.41421356f, 1.68179283f, 2.0f};

static uint64_t synth_base(uint64_t seed, uint32_t tag, uint32_t layer, uint64_t group) {
    return qvo_stream_seed(seed, tag, layer) ^ (group * 0xd1b54a32d192ed03ull);
}

/* Irwin-Hall(4) of the four 16-bit lanes of one splitmix64 draw: mean 131070, sd sqrt(4*(2^32-1)/12). */
static float synth_normal(uint64_t base, uint64_t i) {
    uint64_t st = base + i * 0x9e3779b97f4a7c15ull; /* counter-based splitmix64: draw i of the stream */
    const uint64_t z = qvo_splitmix64(&st);
    const int32_t s = (int32_t)(z & 0xffff) + (int32_t)((z >> 16) & 0xffff) + (int32_t)((z >> 32) & 0xffff) +
                      (int32_t)(z >> 48);
    return (float)(s - 131070) * 2.6428812e-05f; /* 1 / 37837.23 */
}

void qvo_synth_bf16(uint64_t seed, uint32_t tag, uint32_t layer, uint64_t group, size_t rows, uint32_t heads,
                    uint32_t width, int head_scale, uint16_t* out) {
    const uint64_t base = synth_base(seed, tag, layer, group);
    for (size_t r = 0; r < rows; ++r)
        for (uint32_t h = 0; h < heads; ++h) {
            float sc = 1.0f;
            if (head_scale) {
                uint64_t st = base ^ 0x5bd1e995ull;
                st += (r * heads + h) * 0x9e3779b97f4a7c15ull;
                sc = kHeadScale[qvo_splitmix64(&st) % 9];
            }
            for (uint32_t j = 0; j < width; ++j) {
                const size_t e = (r * heads + h) * (size_t)width + j;
                out[e] = qvo_f32_to_bf16(synth_normal(base, e) * sc);
            }
        }
}

void qvo_score_norm(const float* x, size_t n, uint32_t heads, uint32_t width, int negate, double* out) {
    /* prefill.cpp:200-212: sq += double(row[j]) * row[j], j sequential; score = keys ? -sqrt : sqrt */
#pragma omp parallel for schedule(static)
    for (long long i = 0; i < (long long)n; ++i)
        for (uint32_t h = 0; h < heads; ++h) {
            const float* row = x + ((size_t)i * heads + h) * width;
            double sq = 0;
            for (uint32_t j = 0; j < width; ++j) sq += (double)row[j] * row[j];
            const double norm = sqrt(sq);
            out[(size_t)h * n + (size_t)i] = negate ? -norm : norm;
        }
}

void qvo_score_attention(const float* k, size_t n, uint32_t n_h, uint32_t d_h, const float* q, size_t text_count,
                         double* out) {
    /* prefill.cpp:213-230 */
    const size_t d = (size_t)n_h * d_h;
#pragma omp parallel for schedule(static)
    for (long long i = 0; i < (long long)n; ++i) {
        const float* key = k + (size_t)i * d;
        double sum = 0;
        for (size_t t = 0; t < text_count; ++t) {
            const float* qt = q + t * d;
            for (size_t j = 0; j < d; ++j) sum += (double)key[j] * qt[j];
        }
        out[i] = sum / ((double)text_count * n_h);
    }
}

size_t qvo_retained_count(double rho, size_t n) { /* prefill.cpp:235-238 */
    const size_t rounded = (size_t)llround(rho * (double)n);
    size_t k = rounded < 1 ? 1 : rounded;
    return k < n ? k : n;
}

/* (score desc, index asc); -0.0 == +0.0 as in prefill.cpp:245 (`!=` on doubles) */
static const double* g_sort_scores;
static int cmp_better(const void* a, const void* b) {
    const uint32_t ia = *(const uint32_t*)a, ib = *(const uint32_t*)b;
    const double sa = g_sort_scores[ia], sb = g_sort_scores[ib];
    if (sa != sb) return sa > sb ? -1 : 1;
    return ia < ib ? -1 : (ia > ib ? 1 : 0);
}
static int cmp_u32(const void* a, const void* b) {
    const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

size_t qvo_top_k(const double* scores, size_t n, size_t k, uint32_t* out) {
    /* prefill.cpp:240-253 (nth_element + sort restated as a full sort; identical result under a strict order) */
    if (k > n) k = n;
    uint32_t* idx = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
    for (size_t i = 0; i < n; ++i) idx[i] = (uint32_t)i;
    g_sort_scores = scores; /* not reentrant: tests call this single-threaded */
    qsort(idx, n, sizeof(uint32_t), cmp_better);
    qsort(idx, k, sizeof(uint32_t), cmp_u32);
    memcpy(out, idx, k * sizeof(uint32_t));
    free(idx);
    return k;
}

size_t qvo_select_heads(const double* scores, size_t n, uint32_t heads, size_t k, uint32_t* idx) {
    if (k > n) k = n;
    uint32_t* tmp = (uint32_t*)malloc((k ? k : 1) * sizeof(uint32_t));
    for (uint32_t h = 0; h < heads; ++h) {
        qvo_top_k(scores + (size_t)h * n, n, k, tmp);
        for (size_t r = 0; r < k; ++r) idx[r * heads + h] = tmp[r];
    }
    free(tmp);
    return k;
}

void qvo_gather_heads(const float* x, size_t n, uint32_t heads, uint32_t width, const uint32_t* idx, size_t k,
                      float* out) {
    /* prefill.cpp:277-280 per head */
    (void)n;
    for (size_t r = 0; r < k; ++r)
        for (uint32_t h = 0; h < heads; ++h)
            memcpy(out + (r * heads + h) * width, x + ((size_t)idx[r * heads + h] * heads + h) * width,
                   width * sizeof(float));
}

size_t qvo_attention_rows(const float* q, const float* k, const float* v, size_t n, uint32_t n_q, uint32_t n_kv,
                          uint32_t d, double scale, size_t row_begin, size_t row_step, double* o) {
    const uint32_t ratio = n_q / n_kv;
    if (row_step == 0) row_step = 1;
    const long long rows = row_begin < n ? (long long)((n - row_begin + row_step - 1) / row_step) : 0;
#pragma omp parallel
    {
        double* p = (double*)malloc((n ? n : 1) * sizeof(double));
#pragma omp for schedule(dynamic, 4) collapse(2)
        for (long long r = 0; r < rows; ++r)
            for (uint32_t h = 0; h < n_q; ++h) {
                const long long i = (long long)row_begin + r * (long long)row_step;
                const uint32_t hk = h / ratio;
                const float* qi = q + ((size_t)i * n_q + h) * d;
                double m = -INFINITY;
                for (size_t j = 0; j <= (size_t)i; ++j) {
                    const float* kj = k + (j * n_kv + hk) * d;
                    double s = 0;
                    for (uint32_t c = 0; c < d; ++c) s += (double)qi[c] * kj[c];
                    p[j] = s * scale;
                    if (p[j] > m) m = p[j];
                }
                double l = 0;
                for (size_t j = 0; j <= (size_t)i; ++j) {
                    p[j] = exp(p[j] - m);
                    l += p[j];
                }
                double* oi = o + ((size_t)i * n_q + h) * d;
                for (uint32_t c = 0; c < d; ++c) oi[c] = 0;
                for (size_t j = 0; j <= (size_t)i; ++j) {
                    const float* vj = v + (j * n_kv + hk) * d;
                    const double w = p[j] / l;
                    for (uint32_t c = 0; c < d; ++c) oi[c] += w * vj[c];
                }
            }
        free(p);
    }
    return (size_t)rows;
}

void qvo_attention(const float* q, const float* k, const float* v, size_t n, uint32_t n_q, uint32_t n_kv,
                   uint32_t d, double scale, double* o) {
    qvo_attention_rows(q, k, v, n, n_q, n_kv, d, scale, 0, 1, o);
}

void qvo_snapkv_scores(const float* q, const float* k, size_t n, uint32_t n_q, uint32_t n_kv, uint32_t d,
                       uint32_t window, uint32_t pool, double scale, double* out) {
    const uint32_t ratio = n_q / n_kv;
    const size_t w = window < n ? window : n;
    memset(out, 0, (size_t)n_kv * n * sizeof(double));
#pragma omp parallel
    {
        double* p = (double*)malloc((n ? n : 1) * sizeof(double));
#pragma omp for schedule(static)
        for (long long hk = 0; hk < (long long)n_kv; ++hk) {
            double* s = out + (size_t)hk * n;
            for (uint32_t g = 0; g < ratio; ++g) {
                const uint32_t h = (uint32_t)hk * ratio + g;
                for (size_t r = n - w; r < n; ++r) {
                    const float* qr = q + (r * n_q + h) * d;
                    double m = -INFINITY;
                    for (size_t j = 0; j <= r; ++j) {
                        const float* kj = k + (j * n_kv + (size_t)hk) * d;
                        double dot = 0;
                        for (uint32_t c = 0; c < d; ++c) dot += (double)qr[c] * kj[c];
                        p[j] = dot * scale;
                        if (p[j] > m) m = p[j];
                    }
                    double l = 0;
                    for (size_t j = 0; j <= r; ++j) {
                        p[j] = exp(p[j] - m);
                        l += p[j];
                    }
                    for (size_t j = 0; j <= r; ++j) s[j] += p[j] / l;
                }
            }
            if (pool > 1) {
                double* t = (double*)malloc(n * sizeof(double));
                const long long half = pool / 2;
                for (long long j = 0; j < (long long)n; ++j) {
                    double acc = 0;
                    for (long long u = j - half; u <= j + half; ++u)
                        if (u >= 0 && u < (long long)n) acc += s[u];
                    t[j] = acc / pool;
                }
                memcpy(s, t, n * sizeof(double));
                free(t);
            }
        }
        free(p);
    }
}

uint64_t qvo_plan_groups(uint64_t frames, uint32_t fpg, uint32_t tpf, double rho, int64_t* tok_off, int64_t* keep,
                         int64_t* row_off) {
    if (fpg == 0) return 0;
    const uint64_t G = (frames + fpg - 1) / fpg; /* prefill.cpp:325-328 */
    tok_off[0] = 0;
    row_off[0] = 0;
    for (uint64_t g = 0; g < G; ++g) {
        const uint64_t begin = g * fpg; /* prefill.cpp:176-181 */
        const uint64_t end = begin + fpg < frames ? begin + fpg : frames;
        const int64_t n = (int64_t)((end - begin) * tpf);
        tok_off[g + 1] = tok_off[g] + n;
        keep[g] = (int64_t)qvo_retained_count(rho, (size_t)n);
        row_off[g + 1] = row_off[g] + keep[g];
    }
    return G;
}
