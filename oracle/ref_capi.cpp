// TEST INFRASTRUCTURE ONLY — parity checker, never linked into the product.
//
// extern "C" wrapper over the UNMODIFIED reference prefill engine (/root/reference/proj/src/prefill.cpp),
// compiled with -Dqv=qvref (see oracle/Makefile) so every `qv::` below is `qvref::`.  Python tests reach the
// reference through these entry points with ctypes; the C++ parity driver links libqvref.so directly.
//
// Every function returns 0 on success and -1 when the reference threw qv::Error (message via
// qvref_last_error()), so tests can assert the reference's exact error text.
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "qv/prefill.hpp"
#include "qv/synthetic.hpp"

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const qv::Error& e) {
        g_err = e.what();
        return -1;
    } catch (const std::exception& e) {
        g_err = std::string("std: ") + e.what();
        return -2;
    }
}

qv::ModelConfig make_cfg(uint32_t d_model, uint32_t n_h, uint32_t d_h, uint32_t layers, uint32_t tpf,
                         uint32_t text_tokens, uint64_t seed) {
    qv::ModelConfig c;
    c.d_model = d_model;
    c.n_h = n_h;
    c.d_h = d_h;
    c.layers = layers;
    c.tokens_per_frame = tpf;
    c.text_tokens = text_tokens;
    c.seed = seed;
    return c;
}

qv::PruneConfig make_prune(int scorer, double rho) {
    qv::PruneConfig p;
    p.scorer = static_cast<qv::Scorer>(scorer);
    p.rho = rho;
    return p;
}

qv::FrameBuffer make_frames(const uint8_t* pixels, size_t slots, uint32_t width, uint32_t height) {
    qv::FrameBuffer fb(slots, width, height);
    const size_t bytes = fb.slot_bytes();
    for (size_t j = 0; j < slots; ++j) fb.write_slot(j, {pixels + j * bytes, bytes});
    return fb;
}
}  // namespace

extern "C" {

const char* qvref_last_error(void) { return g_err.c_str(); }

// prefill.cpp:192-233
int qvref_score_tokens(const float* k, size_t k_len, const float* v, size_t v_len, size_t token_count,
                       uint32_t n_h, uint32_t d_h, int scorer, const float* q, size_t q_len, double* out) {
    return guard([&] {
        auto s = qv::score_tokens({k, k_len}, {v, v_len}, token_count, n_h, d_h,
                                  static_cast<qv::Scorer>(scorer), {q, q_len});
        std::memcpy(out, s.data(), s.size() * sizeof(double));
    });
}

// prefill.cpp:235-238
size_t qvref_retained_count(double rho, size_t token_count) { return qv::retained_count(rho, token_count); }

// prefill.cpp:240-253
int qvref_top_k_indices(const double* scores, size_t n, size_t k, uint32_t* out, size_t* out_len) {
    return guard([&] {
        auto idx = qv::top_k_indices({scores, n}, k);
        std::memcpy(out, idx.data(), idx.size() * sizeof(uint32_t));
        *out_len = idx.size();
    });
}

// prefill.cpp:255-282.  k_out/v_out must hold k_len/v_len floats, idx_out token_count entries.
int qvref_prune_group(const float* k, size_t k_len, const float* v, size_t v_len, size_t token_count,
                      uint32_t n_h, uint32_t d_h, int scorer, double rho, const float* q, size_t q_len,
                      float* k_out, float* v_out, uint32_t* idx_out, size_t* kept) {
    return guard([&] {
        auto p = qv::prune_group({k, k_len}, {v, v_len}, token_count, n_h, d_h, make_prune(scorer, rho),
                                 {q, q_len});
        std::memcpy(k_out, p.k.data(), p.k.size() * sizeof(float));
        std::memcpy(v_out, p.v.data(), p.v.size() * sizeof(float));
        std::memcpy(idx_out, p.indices.data(), p.indices.size() * sizeof(uint32_t));
        *kept = p.indices.size();
    });
}

// prefill.cpp:325-328
int qvref_group_count(uint64_t total_frames, uint32_t frames_per_group, uint64_t* out) {
    return guard([&] { *out = qv::group_count(total_frames, frames_per_group); });
}

// prefill.cpp:116-121
void qvref_patch_grid(uint32_t tpf, uint32_t* rows, uint32_t* cols) {
    auto [r, c] = qv::StandInModel::patch_grid(tpf);
    *rows = r;
    *cols = c;
}

int qvref_validate_prune(double rho) {
    return guard([&] { make_prune(0, rho).validate(); });
}

int qvref_scorer_from_name(const char* name, int* out) {
    return guard([&] { *out = static_cast<int>(qv::scorer_from_name(name)); });
}

// synthetic.cpp:5-10 / 25-79
uint64_t qvref_splitmix64(uint64_t* state) { return qv::splitmix64(*state); }

void qvref_fill_pattern(int pattern, uint64_t seed, uint64_t index, uint32_t width, uint32_t height,
                        uint8_t* out) {
    qv::fill_pattern(static_cast<qv::Pattern>(pattern), seed, index, width, height,
                     {out, size_t{3} * width * height});
}

// ---- StandInModel (prefill.cpp:96-190) -----------------------------------------------------------
void* qvref_model_create(uint32_t d_model, uint32_t n_h, uint32_t d_h, uint32_t layers, uint32_t tpf,
                         uint32_t text_tokens, uint64_t seed) {
    qv::StandInModel* m = nullptr;
    if (guard([&] { m = new qv::StandInModel(make_cfg(d_model, n_h, d_h, layers, tpf, text_tokens, seed)); }))
        return nullptr;
    return m;
}

void qvref_model_destroy(void* m) { delete static_cast<qv::StandInModel*>(m); }

size_t qvref_model_text_query(void* m, float* out) {
    auto q = static_cast<qv::StandInModel*>(m)->text_query();
    if (out) std::memcpy(out, q.data(), q.size() * sizeof(float));
    return q.size();
}

// K = X W_K, V = X W_V (prefill.cpp:185-190) on caller-provided tokens (token_count x d_model).
int qvref_model_project(void* m, const float* tokens, size_t token_count, uint32_t layer, float* k, float* v) {
    return guard([&] {
        auto* model = static_cast<qv::StandInModel*>(m);
        qv::TokenGroup g;
        g.token_count = token_count;
        g.tokens.assign(tokens, tokens + token_count * model->config().d_model);
        std::vector<float> kk, vv;
        model->project(g, layer, kk, vv);
        std::memcpy(k, kk.data(), kk.size() * sizeof(float));
        std::memcpy(v, vv.data(), vv.size() * sizeof(float));
    });
}

// tokenize (prefill.cpp:170-183): writes all groups' tokens back to back; per-group metadata arrays
// (first_token, frame_begin, frame_end, token_count) must hold group_count(slots, fpg) entries.
int qvref_model_tokenize(void* m, const uint8_t* pixels, size_t slots, uint32_t width, uint32_t height,
                         uint32_t fpg, float* tokens_out, uint64_t* first_token, uint64_t* frame_begin,
                         uint64_t* frame_end, uint64_t* token_count, size_t* n_groups) {
    return guard([&] {
        auto* model = static_cast<qv::StandInModel*>(m);
        qv::FrameBuffer fb = slots ? make_frames(pixels, slots, width, height) : qv::FrameBuffer();
        auto groups = model->tokenize(fb, fpg);
        size_t off = 0;
        for (size_t g = 0; g < groups.size(); ++g) {
            std::memcpy(tokens_out + off, groups[g].tokens.data(), groups[g].tokens.size() * sizeof(float));
            off += groups[g].tokens.size();
            first_token[g] = groups[g].first_token;
            frame_begin[g] = groups[g].frame_begin;
            frame_end[g] = groups[g].frame_end;
            token_count[g] = groups[g].token_count;
        }
        *n_groups = groups.size();
    });
}

// ---- full reference pipeline: tokenize -> prefill (prefill.cpp:316-323) -------------------------
void* qvref_prefill_frames(void* m, const uint8_t* pixels, size_t slots, uint32_t width, uint32_t height,
                           uint32_t fpg, int scorer, double rho) {
    qv::KvCache* out = nullptr;
    if (guard([&] {
            auto* model = static_cast<qv::StandInModel*>(m);
            qv::FrameBuffer fb = make_frames(pixels, slots, width, height);
            auto groups = model->tokenize(fb, fpg);
            out = new qv::KvCache(qv::prefill(*model, groups, make_prune(scorer, rho)));
        }))
        return nullptr;
    return out;
}

void qvref_cache_destroy(void* c) { delete static_cast<qv::KvCache*>(c); }
size_t qvref_cache_layers(void* c) { return static_cast<qv::KvCache*>(c)->layers.size(); }
size_t qvref_cache_rows(void* c, size_t layer) { return static_cast<qv::KvCache*>(c)->layers[layer].origin.size(); }
size_t qvref_cache_groups(void* c) { return static_cast<qv::KvCache*>(c)->retained_per_group.size(); }
uint64_t qvref_cache_tokens_seen(void* c) { return static_cast<qv::KvCache*>(c)->tokens_seen; }
size_t qvref_cache_peak_group_tokens(void* c) { return static_cast<qv::KvCache*>(c)->peak_group_tokens; }
uint64_t qvref_cache_value_bytes(void* c) { return static_cast<qv::KvCache*>(c)->value_bytes(); }

void qvref_cache_copy_layer(void* c, size_t layer, float* k, float* v, uint64_t* origin) {
    const auto& l = static_cast<qv::KvCache*>(c)->layers[layer];
    std::memcpy(k, l.k.data(), l.k.size() * sizeof(float));
    std::memcpy(v, l.v.data(), l.v.size() * sizeof(float));
    std::memcpy(origin, l.origin.data(), l.origin.size() * sizeof(uint64_t));
}

void qvref_cache_retained_per_group(void* c, uint64_t* out) {
    const auto& r = static_cast<qv::KvCache*>(c)->retained_per_group;
    for (size_t i = 0; i < r.size(); ++i) out[i] = r[i];
}

}  // extern "C"
