// extern "C" entry points of include/qvk.h: argument validation with the reference's error texts, the host-side
// group scheduler, and the stream-ordered orchestration of the kernels (score.cu, select.cu, gather.cu,
// attention.cu, snapkv.cu, exact.cu).  No computation of the path happens on the host.
#include <cudaTypedefs.h>

#include <atomic>
#include <cmath>
#include <cstring>
#include <cstdlib>
#include <map>
#include <mutex>
#include <set>
#include <tuple>
#include <string>
#include <vector>

#include "common.cuh"

namespace qvk {

// Trivially destructible, so a qvk call made during process teardown (e.g. a static destructor freeing HBM) can still
// record its error after this thread's thread_local objects with destructors are gone.
thread_local char g_last_error[1024];
void set_error(const std::string& msg) {
    const size_t n = std::min(msg.size(), sizeof(g_last_error) - 1);
    std::memcpy(g_last_error, msg.data(), n);
    g_last_error[n] = '\0';
}

cudaError_t func_attr(const void* func, cudaFuncAttribute attr, int value) {
    static std::mutex mu;
    static std::map<std::tuple<const void*, int, int>, int> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_tuple(func, dev, static_cast<int>(attr));
    auto it = done.find(key);
    if (it != done.end() && it->second >= value) return cudaSuccess;
    e = cudaFuncSetAttribute(func, attr, value);
    if (e == cudaSuccess) done[key] = value;
    return e;
}

cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t stream) {
    // A private pool per device (not the device's default pool, which belongs to the whole process): its release
    // threshold is raised once so freed scratch stays pooled across synchronisations — with the default of 0 every
    // synchronise returns it to the driver and the next call pays a real allocation (~0.4 ms).
    static std::mutex mu;
    static std::map<int, cudaMemPool_t> pools;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    cudaMemPool_t pool;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = pools.find(dev);
        if (it == pools.end()) {
            cudaMemPoolProps props = {};
            props.allocType = cudaMemAllocationTypePinned;
            props.location.type = cudaMemLocationTypeDevice;
            props.location.id = dev;
            e = cudaMemPoolCreate(&pool, &props);
            if (e != cudaSuccess) return e;
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
            pools[dev] = pool;
        } else {
            pool = it->second;
        }
    }
    return cudaMallocFromPoolAsync(p, bytes, pool, stream);
}

thread_local int g_route = -1;

int sm_count() {
    static const int n = [] {
        int dev = 0, v = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
            return kNumSms;
        return v;
    }();
    return n;
}

// SMs the persistent kernels (attention, projection) leave free for work running beside them — the N > 1
// all-gather's NCCL CTAs (qvk_comm_init caps NCCL at QVK_COMM_CTAS CTAs and reserves as many SMs).  A persistent
// grid of one CTA per SM walks a static unit list, so a CTA that has to wait for an SM held by a collective delays
// the whole launch by the collective's duration; with the reservation it never waits.
std::atomic<int> g_reserved_sms{0};

int grid_sms() {
    const int n = sm_count() - g_reserved_sms.load(std::memory_order_relaxed);
    return n < 2 ? 2 : n;
}

}  // namespace qvk

extern "C" int qvk_reserve_sms(int32_t n, int32_t* previous) {
    if (n < 0 || n >= qvk::sm_count()) {
        qvk::set_error("reserve_sms: n must be in [0, SM count)");
        return QVK_E_INVALID;
    }
    const int old = qvk::g_reserved_sms.exchange(n);
    if (previous) *previous = old;
    return QVK_OK;
}

namespace qvk {

int env_knob(const char* name, int def) {
    const char* e = std::getenv(name);
    return e && *e ? std::atoi(e) : def;
}

void* tensor_map_encoder() {
    static void* const fn = [] {
        cudaDriverEntryPointQueryResult q;
        void* ptr = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return static_cast<void*>(nullptr);
        return ptr;
    }();
    return fn;
}

int launch_score(cudaStream_t, const qvk_groups*, int64_t, const void*, const void*, int, int, int, int,
                 const float*, int64_t, int, double*);
int launch_select(cudaStream_t, const qvk_groups*, const double*, int, uint32_t*);
int launch_gather(cudaStream_t, const qvk_groups*, const void*, const void*, int, int, int, const uint32_t*, void*,
                  void*, uint64_t*, int64_t, uint32_t*);
int launch_text_query_sum(cudaStream_t, const float*, int64_t, int, int, int, float*);
int launch_score_dot(cudaStream_t, const qvk_groups*, const void*, int, int, const float*, double, double*);
// lse (optional): the softmax statistics of each group's last lse_window query rows, [group][query head][row] —
// the SnapKV scorer's pass 1, which launch_snapkv then skips.
int launch_attention(cudaStream_t, const qvk_groups*, const void*, const void*, const void*, int, int, int, float,
                     void*, float* lse = nullptr, int lse_window = 0);
int launch_snapkv(cudaStream_t, const qvk_groups*, const void*, const void*, int, int, int, int, int, float,
                  double*, const float* lse = nullptr, int after_attention = 0);
int launch_seeded_matrix(cudaStream_t, uint64_t, uint32_t, uint32_t, size_t, double, float*);
int launch_project_exact(cudaStream_t, const float*, int64_t, int, const float*, int, float*);
int launch_tokenize(cudaStream_t, const uint8_t*, int64_t, uint32_t, uint32_t, uint32_t, uint32_t, uint32_t,
                    const float*, int, void*, int);
int launch_synth_bf16(cudaStream_t, uint64_t, uint32_t, uint32_t, uint64_t, int64_t, int, int, int, void*);
int launch_project_qkv(cudaStream_t, const void*, int64_t, int, const void*, int, int, int, void*, void*, void*,
                       const qvk_groups*, double*);
int launch_decode_attention(cudaStream_t, const void*, int, int, int, int, const void*, const void*, int64_t, float,
                            void*, float*, void*, size_t, size_t*);
int launch_prune_fused_dests(cudaStream_t, const qvk_groups*, const void*, const void*, int, int, int, const double*,
                             double*, uint32_t*, int, void* const*, void* const*, uint64_t* const*, int);
bool prune_fused_supported(const qvk_groups*, int, int, const void*, const void*, const void*, const void*);
bool prune_fused_preferred(const qvk_groups*, int);
int launch_prune_fused(cudaStream_t, const qvk_groups*, const void*, const void*, int, int, int, const double*,
                       double*, uint32_t*, void*, void*, uint64_t*, int);

namespace {

int check_groups(const qvk_groups* g) {
    if (!g) QVK_INVALID("groups: null descriptor");
    if (g->n_groups <= 0) QVK_INVALID("prefill: no token groups");  // prefill.cpp:317
    if (!g->tok_off_d || !g->keep_d || !g->row_off_d) QVK_INVALID("groups: null offset array");
    if (g->max_tokens < 0 || g->total_tokens < 0 || g->total_rows < 0) QVK_INVALID("groups: negative size");
    return QVK_OK;
}

int check_rho(double rho) {
    if (!(rho > 0.0 && rho <= 1.0)) QVK_INVALID("retention ratio must be in (0, 1]");  // prefill.cpp:65-67
    return QVK_OK;
}

size_t retained(double rho, size_t n) {  // prefill.cpp:235-238
    const auto rounded = static_cast<size_t>(std::llround(rho * static_cast<double>(n)));
    return std::min(n, std::max<size_t>(1, rounded));
}

#define QVK_TRY(expr)                 \
    do {                              \
        const int _rc = (expr);       \
        if (_rc != QVK_OK) return _rc; \
    } while (0)

}  // namespace
}  // namespace qvk

using namespace qvk;

extern "C" {

const char* qvk_last_error(void) { return g_last_error; }
int qvk_version(void) { return 2; }
int qvk_last_prune_route(void) { return g_route; }

int qvk_device_count(int* out) {
    QVK_CUDA_CHECK(cudaGetDeviceCount(out));
    return QVK_OK;
}

int qvk_malloc(void** out, size_t bytes) {
    *out = nullptr;
    if (bytes == 0) return QVK_OK;
    QVK_CUDA_CHECK(cudaMalloc(out, bytes));
    return QVK_OK;
}
int qvk_free(void* p) {
    if (p) QVK_CUDA_CHECK(cudaFree(p));
    return QVK_OK;
}
int qvk_memcpy_h2d(void* dst, const void* src, size_t bytes, qvk_stream_t s) {
    if (bytes) QVK_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    return QVK_OK;
}
int qvk_memcpy_d2h(void* dst, const void* src, size_t bytes, qvk_stream_t s) {
    if (bytes) QVK_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
    return QVK_OK;
}
int qvk_stream_sync(qvk_stream_t s) {
    QVK_CUDA_CHECK(cudaStreamSynchronize(s));
    return QVK_OK;
}

// ---- (a1) group scheduler ---------------------------------------------------------------------------------------
int qvk_group_count(uint64_t total_frames, uint32_t fpg, uint64_t* out) {
    if (fpg == 0) QVK_INVALID("frames_per_group must be >= 1");  // prefill.cpp:326
    *out = (total_frames + fpg - 1) / fpg;
    return QVK_OK;
}

size_t qvk_retained_count(double rho, size_t n) { return retained(rho, n); }

int qvk_validate_rho(double rho) { return check_rho(rho); }

int qvk_plan_groups(uint64_t total_frames, uint32_t fpg, uint32_t tpf, double rho, int32_t world,
                    uint64_t* n_groups, int64_t* tok_off, int64_t* keep, int64_t* row_off, int32_t* rank_begin) {
    if (fpg == 0) QVK_INVALID("tokenize: frames_per_group must be >= 1");     // prefill.cpp:173
    if (total_frames == 0) QVK_INVALID("tokenize: empty frame buffer");       // prefill.cpp:172
    if (tpf == 0) QVK_INVALID("model config: dimensions must be positive");   // prefill.cpp:59-60
    QVK_TRY(check_rho(rho));
    if (world < 1) QVK_INVALID("plan: world size must be >= 1");
    const uint64_t G = (total_frames + fpg - 1) / fpg;
    if (n_groups) *n_groups = G;
    if (!tok_off) return QVK_OK;
    tok_off[0] = 0;
    row_off[0] = 0;
    std::vector<double> cost(G);
    double total_cost = 0;
    for (uint64_t g = 0; g < G; ++g) {  // prefill.cpp:176-181: last group may be short
        const uint64_t begin = g * fpg;
        const uint64_t end = std::min<uint64_t>(begin + fpg, total_frames);
        const int64_t n = static_cast<int64_t>((end - begin) * tpf);
        tok_off[g + 1] = tok_off[g] + n;
        keep[g] = static_cast<int64_t>(retained(rho, static_cast<size_t>(n)));
        row_off[g + 1] = row_off[g] + keep[g];
        cost[g] = static_cast<double>(n) * static_cast<double>(n);  // causal attention ~ N^2
        total_cost += cost[g];
    }
    if (rank_begin) {
        // Contiguous blocks balanced by cost: rank r starts at the first group whose cumulative cost reaches
        // r/world of the total; never leave a rank empty while groups remain.
        rank_begin[0] = 0;
        double acc = 0;
        uint64_t g = 0;
        for (int32_t r = 1; r < world; ++r) {
            const double target = total_cost * r / world;
            while (g < G && acc + 0.5 * cost[g] < target) acc += cost[g++];
            const uint64_t min_g = static_cast<uint64_t>(rank_begin[r - 1]) + ((uint64_t)rank_begin[r - 1] < G ? 1 : 0);
            if (g < min_g) {
                for (uint64_t x = g; x < min_g; ++x) acc += cost[x];
                g = min_g;
            }
            rank_begin[r] = static_cast<int32_t>(std::min<uint64_t>(g, G));
        }
        rank_begin[world] = static_cast<int32_t>(G);
    }
    return QVK_OK;
}

// ---- scores ------------------------------------------------------------------------------------------------------
int qvk_score(qvk_stream_t s, const qvk_groups* g, const void* k, const void* v, int dtype, int32_t heads,
              int32_t width, int32_t scorer, const float* tq, int64_t text_count, int32_t n_h, double* scores) {
    QVK_TRY(check_groups(g));
    if (heads <= 0 || width <= 0) QVK_INVALID("model config: dimensions must be positive");
    if (dtype != QVK_F32 && dtype != QVK_BF16) QVK_INVALID("score: unsupported dtype");
    if (scorer == QVK_ATTENTION_SCORE) {
        // prefill.cpp:214-217
        if (!tq || text_count <= 0) QVK_INVALID("attention_score scorer requires a text query");
    } else if (scorer != QVK_KEY_NORM_SMALL && scorer != QVK_VALUE_NORM) {
        QVK_INVALID("score: unknown scorer (use qvk_snapkv_score for SnapKV)");
    }
    return launch_score(s, g, g->total_tokens, k, v, dtype, heads, width, scorer, tq, text_count, n_h, scores);
}

int qvk_snapkv_score(qvk_stream_t s, const qvk_groups* g, const void* q, const void* k, int32_t n_q, int32_t n_kv,
                     int32_t d_h, int32_t window, int32_t pool, float scale, double* scores) {
    QVK_TRY(check_groups(g));
    return launch_snapkv(s, g, q, k, n_q, n_kv, d_h, window, pool, scale, scores);
}

int qvk_snapkv_score_stats(qvk_stream_t s, const qvk_groups* g, const void* q, const void* k, int32_t n_q,
                           int32_t n_kv, int32_t d_h, int32_t window, int32_t pool, float scale, const float* stats,
                           double* scores) {
    QVK_TRY(check_groups(g));
    if (!stats) QVK_INVALID("snapkv: null window statistics");
    return launch_snapkv(s, g, q, k, n_q, n_kv, d_h, window, pool, scale, scores, stats);
}

int qvk_select(qvk_stream_t s, const qvk_groups* g, const double* scores, int32_t heads, uint32_t* idx) {
    QVK_TRY(check_groups(g));
    if (heads <= 0) QVK_INVALID("model config: dimensions must be positive");
    return launch_select(s, g, scores, heads, idx);
}

namespace {
int gather_checked(qvk_stream_t s, const qvk_groups* g, const void* k, const void* v, int dtype, int32_t heads,
                   int32_t width, const uint32_t* idx, void* kc, void* vc, uint64_t* origin, int64_t keep_stride,
                   uint32_t* idx_out) {
    QVK_TRY(check_groups(g));
    if (heads <= 0 || width <= 0) QVK_INVALID("model config: dimensions must be positive");
    if (dtype != QVK_F32 && dtype != QVK_BF16) QVK_INVALID("gather: unsupported dtype");
    return launch_gather(s, g, k, v, dtype, heads, width, idx, kc, vc, origin, keep_stride, idx_out);
}

int check_text(const float* tq, int64_t text_count) {
    if (!tq || text_count <= 0) QVK_INVALID("attention_score scorer requires a text query");  // prefill.cpp:214-215
    return QVK_OK;
}

// GQA attention_score (qvk_score_text): qbar = the text queries pre-summed over text tokens and the query heads of
// each KV head, then the reference's sequential dot product per (token, head) row (score.cu).
int score_text(cudaStream_t s, const qvk_groups* g, const void* k, int n_q, int n_kv, int d_h, int per_head,
               const float* tq, int64_t text_count, float* qbar_ws, double* scores) {
    QVK_TRY(check_text(tq, text_count));
    if (n_q <= 0 || n_kv <= 0 || d_h <= 0) QVK_INVALID("model config: dimensions must be positive");
    if (n_q % n_kv != 0) QVK_INVALID("score: n_q must be a multiple of n_kv");
    float* qb = qbar_ws;
    if (!qb) QVK_CUDA_CHECK(scratch_alloc(reinterpret_cast<void**>(&qb), sizeof(float) * n_kv * d_h, s));
    int rc = launch_text_query_sum(s, tq, text_count, n_q, n_kv, d_h, qb);
    // divisor = T * (query heads averaged over): the reference's double(text_count) * n_h (prefill.cpp:228)
    const double div = static_cast<double>(text_count) * static_cast<double>(per_head ? n_q / n_kv : n_q);
    if (rc == QVK_OK)
        rc = per_head ? launch_score_dot(s, g, k, n_kv, d_h, qb, div, scores)
                      : launch_score_dot(s, g, k, 1, n_kv * d_h, qb, div, scores);
    if (!qbar_ws) cudaFreeAsync(qb, s);
    return rc;
}

// The prune step of one layer (score -> select -> gather into the cache, prefill.cpp:255-282) for every group,
// after the layer's attention.  pre_scores: scores already computed (the key-norm fused into the projection
// epilogue); overlap: the previous kernel on the stream only READS k / v (the attention), so a fused launch may
// start in its tail (PDL).
int layer_prune(cudaStream_t s, const qvk_groups* g, const qvk_layer_params* p, const void* q, const void* k,
                const void* v, const double* pre_scores, double* scores_ws, uint32_t* idx_ws, void* kc, void* vc,
                uint64_t* origin, int overlap, const float* lse = nullptr) {
    const int heads = p->per_head ? p->n_kv : 1;
    const int width = p->per_head ? p->d_h : p->n_kv * p->d_h;
    const int64_t keep_full = static_cast<int64_t>(retained(p->rho, static_cast<size_t>(g->max_tokens)));
    if (origin && !g->first_token_d) QVK_INVALID("gather: origin requested without first_token");
    if (p->rho == 1.0) {  // prefill.cpp:263-270: identity, no scoring
        g_route = 2;
        return launch_gather(s, g, k, v, QVK_BF16, heads, width, nullptr, kc, vc, origin, keep_full, idx_ws);
    }
    const bool fused = prune_fused_supported(g, QVK_BF16, width, k, v, kc, vc) && prune_fused_preferred(g, heads);
    const bool norm = p->scorer == QVK_KEY_NORM_SMALL || p->scorer == QVK_VALUE_NORM;
    if (!pre_scores && norm && fused) {  // score + select + gather in one cluster launch
        g_route = 0;
        return launch_prune_fused(s, g, k, v, heads, width, p->scorer, nullptr, scores_ws, idx_ws, kc, vc, origin,
                                  overlap);
    }
    if (!pre_scores && p->scorer == QVK_SNAPKV && !p->per_head)
        QVK_INVALID("prefill_layer: SnapKV scores are per KV head (set per_head = 1)");
    if (!pre_scores && p->scorer == QVK_ATTENTION_SCORE) QVK_TRY(check_text(p->text_query_d, p->text_count));
    if (!pre_scores && !norm && p->scorer != QVK_ATTENTION_SCORE && p->scorer != QVK_SNAPKV)
        QVK_INVALID("score: unknown scorer");
    double* sc = scores_ws;
    uint32_t* ix = idx_ws;
    if (!pre_scores && !sc)
        QVK_CUDA_CHECK(scratch_alloc(reinterpret_cast<void**>(&sc),
                                     sizeof(double) * std::max<int64_t>(1, g->total_tokens * heads), s));
    int rc = QVK_OK;
    if (!pre_scores) {
        if (p->scorer == QVK_SNAPKV)
            rc = launch_snapkv(s, g, q, k, p->n_q, p->n_kv, p->d_h, p->snap_window, p->snap_pool, p->scale, sc, lse,
                               lse != nullptr);  // right behind the attention that writes lse: PDL
        else if (p->scorer == QVK_ATTENTION_SCORE)
            rc = score_text(s, g, k, p->n_q, p->n_kv, p->d_h, p->per_head, p->text_query_d, p->text_count, nullptr,
                            sc);
        else
            rc = launch_score(s, g, g->total_tokens, k, v, QVK_BF16, heads, width, p->scorer, nullptr, 0, 1, sc);
    }
    const double* scores = pre_scores ? pre_scores : sc;
    if (rc == QVK_OK && fused) {  // select + gather fused on the given scores
        g_route = 3;
        rc = launch_prune_fused(s, g, k, v, heads, width, QVK_SNAPKV, scores, nullptr, idx_ws, kc, vc, origin,
                                pre_scores ? overlap : 0);
    } else if (rc == QVK_OK) {
        g_route = 1;
        if (!ix)
            QVK_CUDA_CHECK(scratch_alloc(reinterpret_cast<void**>(&ix),
                                         sizeof(uint32_t) * std::max<int64_t>(1, g->total_rows * heads), s));
        rc = launch_select(s, g, scores, heads, ix);
        if (rc == QVK_OK) rc = launch_gather(s, g, k, v, QVK_BF16, heads, width, ix, kc, vc, origin, keep_full, nullptr);
        if (!idx_ws) cudaFreeAsync(ix, s);
    }
    if (!pre_scores && !scores_ws) cudaFreeAsync(sc, s);
    return rc;
}
// SnapKV's pass 1 (the window rows' softmax statistics) comes out of the layer's attention kernel when the layer
// prunes with SnapKV scores: a window-statistics buffer of n_groups * n_q * window floats (lse_ws, or scratch).
bool snap_from_attention(const qvk_layer_params* p) {
    static const int on = env_knob("QVK_SNAPKV_LSE", 1);
    return on && p->scorer == QVK_SNAPKV && p->per_head && p->rho != 1.0 && p->d_h == 128 && p->snap_window > 0;
}
size_t snap_lse_bytes(const qvk_groups* g, const qvk_layer_params* p) {
    return sizeof(float) * std::max<int64_t>(1, static_cast<int64_t>(g->n_groups) * p->n_q * p->snap_window);
}

// attention -> prune of one layer (q / k / v already on the device)
int layer_from_qkv(cudaStream_t s, const qvk_groups* g, const qvk_layer_params* p, const void* q, const void* k,
                   const void* v, void* o, const double* pre_scores, double* scores_ws, uint32_t* idx_ws, void* kc,
                   void* vc, uint64_t* origin, float* lse_ws) {
    float* lse = nullptr;
    if (snap_from_attention(p)) {
        lse = lse_ws;
        if (!lse) QVK_CUDA_CHECK(scratch_alloc(reinterpret_cast<void**>(&lse), snap_lse_bytes(g, p), s));
    }
    int rc = launch_attention(s, g, q, k, v, p->n_q, p->n_kv, p->d_h, p->scale, o, lse, lse ? p->snap_window : 0);
    // overlap = 1: the fused prune only reads K / V, so its CTAs may take the SMs the attention grid releases
    if (rc == QVK_OK) rc = layer_prune(s, g, p, q, k, v, pre_scores, scores_ws, idx_ws, kc, vc, origin, 1, lse);
    if (lse && !lse_ws) cudaFreeAsync(lse, s);
    return rc;
}
}  // namespace

int qvk_gather(qvk_stream_t s, const qvk_groups* g, const void* k, const void* v, int dtype, int32_t heads,
               int32_t width, const uint32_t* idx, void* kc, void* vc, uint64_t* origin) {
    return gather_checked(s, g, k, v, dtype, heads, width, idx, kc, vc, origin, 0, nullptr);
}

int qvk_select_gather(qvk_stream_t s, const qvk_groups* g, const double* scores, const void* k, const void* v,
                      int dtype, int32_t heads, int32_t width, uint32_t* idx, void* kc, void* vc, uint64_t* origin) {
    QVK_TRY(check_groups(g));
    if (heads <= 0 || width <= 0) QVK_INVALID("model config: dimensions must be positive");
    if (dtype != QVK_F32 && dtype != QVK_BF16) QVK_INVALID("gather: unsupported dtype");
    if (origin && !g->first_token_d) QVK_INVALID("gather: origin requested without first_token");
    if (prune_fused_supported(g, dtype, width, k, v, kc, vc) && prune_fused_preferred(g, heads)) {
        g_route = 3;
        return launch_prune_fused(s, g, k, v, heads, width, QVK_SNAPKV, scores, nullptr, idx, kc, vc, origin, 0);
    }
    g_route = 1;
    uint32_t* ix = idx;
    if (!ix) QVK_CUDA_CHECK(scratch_alloc(reinterpret_cast<void**>(&ix),
                                            sizeof(uint32_t) * std::max<int64_t>(1, g->total_rows * heads), s));
    int rc = launch_select(s, g, scores, heads, ix);
    if (rc == QVK_OK) rc = launch_gather(s, g, k, v, dtype, heads, width, ix, kc, vc, origin, 0, nullptr);
    if (!idx) cudaFreeAsync(ix, s);
    return rc;
}

int qvk_prune(qvk_stream_t s, const qvk_groups* g, const void* k, const void* v, int dtype, int32_t heads,
              int32_t width, int32_t scorer, double rho, const float* tq, int64_t text_count, int32_t n_h,
              double* scores_ws, uint32_t* idx_ws, void* kc, void* vc, uint64_t* origin) {
    QVK_TRY(check_rho(rho));  // prefill.cpp:258, validated before anything else
    QVK_TRY(check_groups(g));
    const int64_t keep_full = static_cast<int64_t>(retained(rho, static_cast<size_t>(g->max_tokens)));
    if (rho == 1.0) {  // prefill.cpp:263-270: identity, no scoring, no shape check
        g_route = 2;
        return gather_checked(s, g, k, v, dtype, heads, width, nullptr, kc, vc, origin, keep_full, idx_ws);
    }
    if (origin && !g->first_token_d) QVK_INVALID("gather: origin requested without first_token");
    if ((scorer == QVK_KEY_NORM_SMALL || scorer == QVK_VALUE_NORM) && heads > 0 && width > 0 &&
        prune_fused_supported(g, dtype, width, k, v, kc, vc) && prune_fused_preferred(g, heads)) {
        // score -> select -> gather in one cluster launch (prune_fused.cu); workspaces receive scores / idx
        g_route = 0;
        return launch_prune_fused(s, g, k, v, heads, width, scorer, nullptr, scores_ws, idx_ws, kc, vc, origin, 0);
    }
    g_route = 1;
    double* sc = scores_ws;
    uint32_t* ix = idx_ws;
    if (!sc) QVK_CUDA_CHECK(scratch_alloc(reinterpret_cast<void**>(&sc),
                                            sizeof(double) * std::max<int64_t>(1, g->total_tokens * heads), s));
    if (!ix) QVK_CUDA_CHECK(scratch_alloc(reinterpret_cast<void**>(&ix),
                                            sizeof(uint32_t) * std::max<int64_t>(1, g->total_rows * heads), s));
    int rc = qvk_score(s, g, k, v, dtype, heads, width, scorer, tq, text_count, n_h, sc);
    if (rc == QVK_OK) rc = qvk_select(s, g, sc, heads, ix);
    if (rc == QVK_OK) rc = gather_checked(s, g, k, v, dtype, heads, width, ix, kc, vc, origin, keep_full, nullptr);
    if (!scores_ws) cudaFreeAsync(sc, s);
    if (!idx_ws) cudaFreeAsync(ix, s);
    return rc;
}

int qvk_text_query_sum(qvk_stream_t s, const float* tq, int64_t text_count, int32_t n_q, int32_t n_kv, int32_t d_h,
                       float* qbar) {
    QVK_TRY(check_text(tq, text_count));
    if (n_q <= 0 || n_kv <= 0 || d_h <= 0) QVK_INVALID("model config: dimensions must be positive");
    if (n_q % n_kv != 0) QVK_INVALID("score: n_q must be a multiple of n_kv");
    if (!qbar) QVK_INVALID("score: null qbar output");
    return launch_text_query_sum(s, tq, text_count, n_q, n_kv, d_h, qbar);
}

int qvk_score_text(qvk_stream_t s, const qvk_groups* g, const void* k, int32_t n_q, int32_t n_kv, int32_t d_h,
                   int32_t per_head, const float* tq, int64_t text_count, float* qbar_ws, double* scores) {
    QVK_TRY(check_groups(g));
    return score_text(s, g, k, n_q, n_kv, d_h, per_head, tq, text_count, qbar_ws, scores);
}

int qvk_attention(qvk_stream_t s, const qvk_groups* g, const void* q, const void* k, const void* v, int32_t n_q,
                  int32_t n_kv, int32_t d_h, float scale, void* o) {
    QVK_TRY(check_groups(g));
    return launch_attention(s, g, q, k, v, n_q, n_kv, d_h, scale, o);
}

int qvk_attention_window_stats(qvk_stream_t s, const qvk_groups* g, const void* q, const void* k, const void* v,
                               int32_t n_q, int32_t n_kv, int32_t d_h, float scale, void* o, int32_t window,
                               float* stats) {
    QVK_TRY(check_groups(g));
    if (!stats || window <= 0) QVK_INVALID("attention: window statistics need a buffer and a window >= 1");
    if (d_h != 128) {
        set_error("attention: window statistics need head_dim 128");
        return QVK_E_UNSUPPORTED;
    }
    return launch_attention(s, g, q, k, v, n_q, n_kv, d_h, scale, o, stats, window);
}

static int prefill_layer_impl(qvk_stream_t s, const qvk_groups* g, const qvk_layer_params* p, const void* q,
                              const void* k, const void* v, void* o, double* scores_ws, uint32_t* idx_ws, void* kc,
                              void* vc, uint64_t* origin, float* lse_ws) {
    if (!p) QVK_INVALID("prefill_layer: null params");
    QVK_TRY(check_rho(p->rho));
    QVK_TRY(check_groups(g));
    if (origin && !g->first_token_d) QVK_INVALID("gather: origin requested without first_token");
    return layer_from_qkv(s, g, p, q, k, v, o, nullptr, scores_ws, idx_ws, kc, vc, origin, lse_ws);
}

int qvk_prefill_layer(qvk_stream_t s, const qvk_groups* g, const qvk_layer_params* p, const void* q,
                      const void* k, const void* v, void* o, double* scores_ws, uint32_t* idx_ws, void* kc, void* vc,
                      uint64_t* origin) {
    return prefill_layer_impl(s, g, p, q, k, v, o, scores_ws, idx_ws, kc, vc, origin, nullptr);
}

int qvk_project_qkv(qvk_stream_t s, const void* x, int64_t tokens, int32_t d_model, const void* w, int32_t n_q,
                    int32_t n_kv, int32_t d_h, void* q, void* k, void* v, const qvk_groups* g, double* scores) {
    if (g) QVK_TRY(check_groups(g));
    if (n_q > 0 && n_kv > 0 && n_q % n_kv != 0) QVK_INVALID("project: n_q must be a multiple of n_kv");
    return launch_project_qkv(s, x, tokens, d_model, w, n_q, n_kv, d_h, q, k, v, g, scores);
}

static int prefill_layer_x_impl(qvk_stream_t s, const qvk_groups* g, const qvk_layer_params* p, const void* x,
                                int32_t d_model, const void* w, void* q, void* k, void* v, void* o, double* scores_ws,
                                uint32_t* idx_ws, void* kc, void* vc, uint64_t* origin, float* lse_ws) {
    if (!p) QVK_INVALID("prefill_layer: null params");
    QVK_TRY(check_rho(p->rho));
    QVK_TRY(check_groups(g));
    if (!scores_ws) QVK_INVALID("prefill_layer_x: scores workspace required");
    if (origin && !g->first_token_d) QVK_INVALID("gather: origin requested without first_token");
    const bool fused_norm = p->scorer == QVK_KEY_NORM_SMALL && p->per_head && p->rho != 1.0;
    QVK_TRY(launch_project_qkv(s, x, g->total_tokens, d_model, w, p->n_q, p->n_kv, p->d_h, q, k, v, g,
                               fused_norm ? scores_ws : nullptr));
    // key-norm scores came from the projection epilogue: select + gather only, in the attention's tail
    return layer_from_qkv(s, g, p, q, k, v, o, fused_norm ? scores_ws : nullptr, scores_ws, idx_ws, kc, vc, origin,
                          lse_ws);
}

int qvk_prefill_layer_x(qvk_stream_t s, const qvk_groups* g, const qvk_layer_params* p, const void* x,
                        int32_t d_model, const void* w, void* q, void* k, void* v, void* o, double* scores_ws,
                        uint32_t* idx_ws, void* kc, void* vc, uint64_t* origin) {
    return prefill_layer_x_impl(s, g, p, x, d_model, w, q, k, v, o, scores_ws, idx_ws, kc, vc, origin, nullptr);
}

int qvk_decode_workspace(int32_t n_tq, int32_t n_q, int32_t n_kv, int32_t d_h, int64_t rows, size_t* bytes) {
    if (!bytes) QVK_INVALID("decode_workspace: null output");
    // size query: no tensors are touched (aligned dummy pointers pass the checks)
    void* const dummy = reinterpret_cast<void*>(uintptr_t(256));
    return launch_decode_attention(nullptr, dummy, n_tq, n_q, n_kv, d_h, dummy, dummy, rows, 1.f, dummy, nullptr,
                                   nullptr, 0, bytes);
}

int qvk_decode_attention(qvk_stream_t s, const void* q, int32_t n_tq, int32_t n_q, int32_t n_kv, int32_t d_h,
                         const void* kc, const void* vc, int64_t rows, float scale, void* o, float* lse, void* ws,
                         size_t ws_bytes) {
    if (!ws) QVK_INVALID("decode_attention: workspace required");
    return launch_decode_attention(s, q, n_tq, n_q, n_kv, d_h, kc, vc, rows, scale, o, lse, ws, ws_bytes, nullptr);
}

// ---- multi-GPU: peer caches ---------------------------------------------------------------------------------------
int qvk_ipc_get_handle(const void* ptr, void* handle_out, uint64_t* offset_out) {
    if (!ptr || !handle_out || !offset_out) QVK_INVALID("ipc: null argument");
    static const PFN_cuMemGetAddressRange_v3020 range = [] {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(fn);
    }();
    if (!range) QVK_INVALID("ipc: cuMemGetAddressRange unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS) QVK_INVALID("ipc: not device memory");
    cudaIpcMemHandle_t h;
    QVK_CUDA_CHECK(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    std::memcpy(handle_out, &h, sizeof(h));
    *offset_out = reinterpret_cast<uint64_t>(ptr) - static_cast<uint64_t>(base);
    return QVK_OK;
}

int qvk_ipc_open(const void* handle, void** base_out) {
    if (!handle || !base_out) QVK_INVALID("ipc: null argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    QVK_CUDA_CHECK(cudaIpcOpenMemHandle(base_out, h, cudaIpcMemLazyEnablePeerAccess));
    return QVK_OK;
}

int qvk_ipc_close(void* base) {
    if (base) QVK_CUDA_CHECK(cudaIpcCloseMemHandle(base));
    return QVK_OK;
}

int qvk_prune_dests(qvk_stream_t s, const qvk_groups* g, const void* k, const void* v, int32_t heads, int32_t width,
                    int32_t scorer, double rho, double* scores_ws, uint32_t* idx_ws, int32_t n_dest,
                    void* const* kc, void* const* vc, uint64_t* const* origin) {
    QVK_TRY(check_rho(rho));
    QVK_TRY(check_groups(g));
    if (heads <= 0 || width <= 0) QVK_INVALID("model config: dimensions must be positive");
    if (!kc || !vc || n_dest < 1) QVK_INVALID("prune: no cache destinations");
    if (origin && !g->first_token_d) QVK_INVALID("gather: origin requested without first_token");
    if (rho == 1.0 || (scorer != QVK_KEY_NORM_SMALL && scorer != QVK_VALUE_NORM) ||
        !prune_fused_supported(g, QVK_BF16, width, k, v, kc[0], vc[0])) {
        set_error("prune_dests: needs rho < 1, a norm scorer and bf16 rows of 64/128/256/512");
        return QVK_E_UNSUPPORTED;
    }
    g_route = 0;
    return launch_prune_fused_dests(s, g, k, v, heads, width, scorer, nullptr, scores_ws, idx_ws, n_dest, kc, vc,
                                    origin, 0);
}

int qvk_prefill_layer_dests(qvk_stream_t s, const qvk_groups* g, const qvk_layer_params* p, const void* q,
                            const void* k, const void* v, void* o, double* scores_ws, uint32_t* idx_ws,
                            int32_t n_dest, void* const* kc, void* const* vc, uint64_t* const* origin) {
    if (!p) QVK_INVALID("prefill_layer: null params");
    QVK_TRY(check_rho(p->rho));
    QVK_TRY(check_groups(g));
    if (!kc || !vc || n_dest < 1) QVK_INVALID("prune: no cache destinations");
    if (origin && !g->first_token_d) QVK_INVALID("gather: origin requested without first_token");
    const int heads = p->per_head ? p->n_kv : 1;
    const int width = p->per_head ? p->d_h : p->n_kv * p->d_h;
    if (p->rho == 1.0 || (p->scorer != QVK_KEY_NORM_SMALL && p->scorer != QVK_VALUE_NORM) ||
        !prune_fused_supported(g, QVK_BF16, width, k, v, kc[0], vc[0])) {
        set_error("prefill_layer_dests: needs rho < 1, a norm scorer and bf16 rows of 64/128/256/512");
        return QVK_E_UNSUPPORTED;
    }
    QVK_TRY(launch_attention(s, g, q, k, v, p->n_q, p->n_kv, p->d_h, p->scale, o));
    g_route = 0;
    return launch_prune_fused_dests(s, g, k, v, heads, width, p->scorer, nullptr, scores_ws, idx_ws, n_dest, kc, vc,
                                    origin, 1);
}

// ---- stand-in model pieces --------------------------------------------------------------------------------------
int qvk_seeded_matrix(qvk_stream_t s, uint64_t seed, uint32_t tag, uint32_t layer, size_t count, double scale,
                      float* out) {
    return launch_seeded_matrix(s, seed, tag, layer, count, scale, out);
}

int qvk_project_exact(qvk_stream_t s, const float* x, int64_t rows, int32_t d_in, const float* w, int32_t d_out,
                      float* out) {
    if (rows < 0 || d_in <= 0 || d_out <= 0) QVK_INVALID("model config: dimensions must be positive");
    return launch_project_exact(s, x, rows, d_in, w, d_out, out);
}

void qvk_patch_grid(uint32_t tpf, uint32_t* rows, uint32_t* cols) {  // prefill.cpp:116-121
    uint32_t r = 1;
    for (uint32_t x = 1; static_cast<uint64_t>(x) * x <= tpf; ++x)
        if (tpf % x == 0) r = x;
    *rows = r;
    *cols = tpf / r;
}

int qvk_tokenize(qvk_stream_t s, const uint8_t* frames, int64_t n_frames, uint32_t width, uint32_t height,
                 uint32_t tpf, const float* embed, int32_t d_model, float* tokens) {
    if (tpf == 0 || d_model <= 0) QVK_INVALID("model config: dimensions must be positive");
    uint32_t gr, gc;
    qvk_patch_grid(tpf, &gr, &gc);
    if (height % gr != 0 || width % gc != 0)  // prefill.cpp:128-129
        QVK_INVALID("tokenize: frame size not divisible into the patch grid");
    return launch_tokenize(s, frames, n_frames, width, height, tpf, gr, gc, embed, d_model, tokens, 0);
}

int qvk_tokenize_bf16(qvk_stream_t s, const uint8_t* frames, int64_t n_frames, uint32_t width, uint32_t height,
                      uint32_t tpf, const float* embed, int32_t d_model, void* tokens) {
    if (tpf == 0 || d_model <= 0) QVK_INVALID("model config: dimensions must be positive");
    uint32_t gr, gc;
    qvk_patch_grid(tpf, &gr, &gc);
    if (height % gr != 0 || width % gc != 0)  // prefill.cpp:128-129
        QVK_INVALID("tokenize: frame size not divisible into the patch grid");
    return launch_tokenize(s, frames, n_frames, width, height, tpf, gr, gc, embed, d_model, tokens, 1);
}

int qvk_synth_bf16(qvk_stream_t s, uint64_t seed, uint32_t tag, uint32_t layer, uint64_t group, int64_t rows,
                   int32_t heads, int32_t width, int32_t head_scale, void* out) {
    return launch_synth_bf16(s, seed, tag, layer, group, rows, heads, width, head_scale, out);
}

}  // extern "C"

// ---- per-model / per-video context (include/qvk.h qvk_ctx_*) ------------------------------------------------------
struct qvk_ctx_st {
    qvk_layer_params p{};
    qvk_groups g{};
    int device = 0;
    void* arrays = nullptr;   // tok_off | keep | row_off | first_token (int64 / uint64)
    double* scores = nullptr; // n_kv * total_tokens
    uint32_t* idx = nullptr;  // total_rows * n_kv
    float* lse = nullptr;     // SnapKV window statistics (snap_lse_bytes), when the scorer is SnapKV
};

extern "C" {

int qvk_ctx_create(qvk_ctx_t* out, const qvk_layer_params* p, int32_t n_groups, const int64_t* tok_off,
                   const uint64_t* first_token) {
    if (!out || !p || !tok_off) QVK_INVALID("ctx: null argument");
    *out = nullptr;
    if (n_groups <= 0) QVK_INVALID("prefill: no token groups");  // prefill.cpp:317
    QVK_TRY(check_rho(p->rho));
    if (p->n_q <= 0 || p->n_kv <= 0 || p->d_h <= 0) QVK_INVALID("model config: dimensions must be positive");
    const int G = n_groups;
    std::vector<int64_t> host(4 * static_cast<size_t>(G) + 2);
    int64_t* h_tok = host.data();
    int64_t* h_keep = h_tok + G + 1;
    int64_t* h_row = h_keep + G;
    int64_t* h_first = h_row + G + 1;
    int64_t mx = 0;
    h_row[0] = 0;
    for (int i = 0; i <= G; ++i) h_tok[i] = tok_off[i];
    for (int i = 0; i < G; ++i) {
        const int64_t n = tok_off[i + 1] - tok_off[i];
        if (n < 0) QVK_INVALID("ctx: token offsets must be ascending");
        h_keep[i] = static_cast<int64_t>(retained(p->rho, static_cast<size_t>(n)));
        h_row[i + 1] = h_row[i] + h_keep[i];
        h_first[i] = first_token ? static_cast<int64_t>(first_token[i]) : tok_off[i];
        mx = std::max(mx, n);
    }
    auto* c = new qvk_ctx_st;
    c->p = *p;
    cudaGetDevice(&c->device);
    const int heads = p->per_head ? p->n_kv : 1;
    const int64_t T = h_tok[G] - h_tok[0], R = h_row[G];
    if (h_tok[0] != 0) {
        delete c;
        QVK_INVALID("ctx: tok_off[0] must be 0");
    }
    auto fail = [&](cudaError_t e) {
        set_error(std::string("CUDA error: ") + cudaGetErrorString(e) + " in qvk_ctx_create");
        cudaFree(c->arrays);
        cudaFree(c->scores);
        cudaFree(c->idx);
        cudaFree(c->lse);
        delete c;
        return QVK_E_CUDA;
    };
    cudaError_t e;
    if ((e = cudaMalloc(&c->arrays, host.size() * sizeof(int64_t))) != cudaSuccess) return fail(e);
    if ((e = cudaMemcpy(c->arrays, host.data(), host.size() * sizeof(int64_t), cudaMemcpyHostToDevice)) != cudaSuccess)
        return fail(e);
    if ((e = cudaMalloc(reinterpret_cast<void**>(&c->scores), sizeof(double) * std::max<int64_t>(1, T * heads))) !=
        cudaSuccess)
        return fail(e);
    if ((e = cudaMalloc(reinterpret_cast<void**>(&c->idx), sizeof(uint32_t) * std::max<int64_t>(1, R * heads))) !=
        cudaSuccess)
        return fail(e);
    const int64_t* base = static_cast<const int64_t*>(c->arrays);
    c->g.n_groups = G;
    if (snap_from_attention(p) &&
        (e = cudaMalloc(reinterpret_cast<void**>(&c->lse), snap_lse_bytes(&c->g, p))) != cudaSuccess)
        return fail(e);
    c->g.max_tokens = mx;
    c->g.total_tokens = T;
    c->g.total_rows = R;
    c->g.tok_off_d = base;
    c->g.keep_d = base + G + 1;
    c->g.row_off_d = base + 2 * G + 1;
    c->g.first_token_d = reinterpret_cast<const uint64_t*>(base + 3 * G + 2);
    *out = c;
    return QVK_OK;
}

int qvk_ctx_groups(qvk_ctx_t c, qvk_groups* out) {
    if (!c || !out) QVK_INVALID("ctx: null argument");
    *out = c->g;
    return QVK_OK;
}

int qvk_ctx_prefill_layer(qvk_ctx_t c, qvk_stream_t s, const void* q, const void* k, const void* v, void* o,
                          void* kc, void* vc, uint64_t* origin) {
    if (!c) QVK_INVALID("ctx: null argument");
    return prefill_layer_impl(s, &c->g, &c->p, q, k, v, o, c->scores, c->idx, kc, vc, origin, c->lse);
}

int qvk_ctx_prefill_layer_x(qvk_ctx_t c, qvk_stream_t s, const void* x, int32_t d_model, const void* w, void* q,
                            void* k, void* v, void* o, void* kc, void* vc, uint64_t* origin) {
    if (!c) QVK_INVALID("ctx: null argument");
    return prefill_layer_x_impl(s, &c->g, &c->p, x, d_model, w, q, k, v, o, c->scores, c->idx, kc, vc, origin,
                                c->lse);
}

int qvk_ctx_destroy(qvk_ctx_t c) {
    if (!c) return QVK_OK;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(c->device);
    cudaFree(c->arrays);
    cudaFree(c->scores);
    cudaFree(c->idx);
    cudaFree(c->lse);
    cudaSetDevice(cur);
    delete c;
    return QVK_OK;
}

}  // extern "C"
