// TEST INFRASTRUCTURE — end-to-end parity of the drop-in qv:: API (libqv_prefill.so -> libqvk.so, on the GPU)
// against the UNMODIFIED reference (oracle/_ref/libqvref.so through oracle/ref_capi.cpp).
//
//   parity_driver pipeline <pattern> <seed> <frames> <w> <h> <d_model> <n_h> <d_h> <layers> <tpf> <text> <fpg>
//                          <scorer> <rho>
//       synth frames (reference fill_pattern) -> StandInModel -> tokenize -> prefill, on both sides; prints one
//       JSON line with bitwise comparisons of tokens, text query, every layer's K/V/origin and the cache stats.
//   parity_driver errors
//       drives the documented misuse cases through both APIs and prints each pair of qv::Error messages.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "qv/prefill.hpp"
#include "qv/synthetic.hpp"
#include "qv_pipeline.hpp"

extern "C" {
const char* qvref_last_error(void);
void qvref_fill_pattern(int, uint64_t, uint64_t, uint32_t, uint32_t, uint8_t*);
void* qvref_model_create(uint32_t, uint32_t, uint32_t, uint32_t, uint32_t, uint32_t, uint64_t);
void qvref_model_destroy(void*);
size_t qvref_model_text_query(void*, float*);
int qvref_model_tokenize(void*, const uint8_t*, size_t, uint32_t, uint32_t, uint32_t, float*, uint64_t*, uint64_t*,
                         uint64_t*, uint64_t*, size_t*);
void* qvref_prefill_frames(void*, const uint8_t*, size_t, uint32_t, uint32_t, uint32_t, int, double);
void qvref_cache_destroy(void*);
size_t qvref_cache_layers(void*);
size_t qvref_cache_rows(void*, size_t);
size_t qvref_cache_groups(void*);
uint64_t qvref_cache_tokens_seen(void*);
size_t qvref_cache_peak_group_tokens(void*);
uint64_t qvref_cache_value_bytes(void*);
void qvref_cache_copy_layer(void*, size_t, float*, float*, uint64_t*);
void qvref_cache_retained_per_group(void*, uint64_t*);
int qvref_score_tokens(const float*, size_t, const float*, size_t, size_t, uint32_t, uint32_t, int, const float*,
                       size_t, double*);
int qvref_prune_group(const float*, size_t, const float*, size_t, size_t, uint32_t, uint32_t, int, double,
                      const float*, size_t, float*, float*, uint32_t*, size_t*);
int qvref_group_count(uint64_t, uint32_t, uint64_t*);
}

namespace {

template <class T>
bool same_bits(const std::vector<T>& a, const T* b, size_t n) {
    return a.size() == n && (n == 0 || std::memcmp(a.data(), b, n * sizeof(T)) == 0);
}

int pipeline(char** a) {
    const int pattern = std::stoi(a[0]);
    const uint64_t seed = std::stoull(a[1]);
    const size_t frames = std::stoull(a[2]);
    const uint32_t w = std::stoul(a[3]), h = std::stoul(a[4]);
    qv::ModelConfig cfg;
    cfg.d_model = std::stoul(a[5]);
    cfg.n_h = std::stoul(a[6]);
    cfg.d_h = std::stoul(a[7]);
    cfg.layers = std::stoul(a[8]);
    cfg.tokens_per_frame = std::stoul(a[9]);
    cfg.text_tokens = std::stoul(a[10]);
    cfg.seed = seed;
    const uint32_t fpg = std::stoul(a[11]);
    qv::PruneConfig prune;
    prune.scorer = qv::scorer_from_name(a[12]);
    prune.rho = std::stod(a[13]);

    qv::FrameBuffer fb(frames, w, h);
    std::vector<uint8_t> pixels(frames * fb.slot_bytes());
    for (size_t f = 0; f < frames; ++f) {
        qvref_fill_pattern(pattern, seed, f, w, h, pixels.data() + f * fb.slot_bytes());
        fb.write_slot(f, {pixels.data() + f * fb.slot_bytes(), fb.slot_bytes()});
    }

    // drop-in (GPU); the timed part is tokenize + prefill, the same scope as the reference call timed below
    qv::StandInModel model(cfg);
    const auto t0 = std::chrono::steady_clock::now();
    const auto groups = model.tokenize(fb, fpg);
    const qv::KvCache cache = qv::prefill(model, groups, prune);
    const double dropin_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();

    // reference (CPU)
    void* ref = qvref_model_create(cfg.d_model, cfg.n_h, cfg.d_h, cfg.layers, cfg.tokens_per_frame,
                                   cfg.text_tokens, seed);
    std::vector<float> ref_q(size_t{cfg.text_tokens} * cfg.d_model);
    qvref_model_text_query(ref, ref_q.data());
    const size_t n_tok = frames * cfg.tokens_per_frame;
    std::vector<float> ref_tok(n_tok * cfg.d_model);
    std::vector<uint64_t> ft(groups.size() + 1), fbg(groups.size() + 1), fe(groups.size() + 1), tc(groups.size() + 1);
    size_t n_groups = 0;
    qvref_model_tokenize(ref, pixels.data(), frames, w, h, fpg, ref_tok.data(), ft.data(), fbg.data(), fe.data(),
                         tc.data(), &n_groups);
    bool tokens_equal = n_groups == groups.size();
    size_t off = 0;
    for (size_t g = 0; tokens_equal && g < groups.size(); ++g) {
        tokens_equal = same_bits(groups[g].tokens, ref_tok.data() + off, size_t(tc[g]) * cfg.d_model) &&
                       groups[g].first_token == ft[g] && groups[g].frame_begin == fbg[g] &&
                       groups[g].frame_end == fe[g] && groups[g].token_count == tc[g];
        off += size_t(tc[g]) * cfg.d_model;
    }
    const auto q = model.text_query();
    const bool query_equal = same_bits(std::vector<float>(q.begin(), q.end()), ref_q.data(), ref_q.size());

    const auto t1 = std::chrono::steady_clock::now();
    void* rc = qvref_prefill_frames(ref, pixels.data(), frames, w, h, fpg, static_cast<int>(prune.scorer), prune.rho);
    const double ref_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count();
    bool cache_equal = rc && qvref_cache_layers(rc) == cache.layers.size();
    size_t rows = 0;
    int first_bad_layer = -1;
    for (size_t l = 0; cache_equal && l < cache.layers.size(); ++l) {
        const size_t r = qvref_cache_rows(rc, l);
        const size_t d = cfg.d_model;
        std::vector<float> k(r * d), v(r * d);
        std::vector<uint64_t> o(r);
        qvref_cache_copy_layer(rc, l, k.data(), v.data(), o.data());
        const bool ok = same_bits(cache.layers[l].k, k.data(), r * d) && same_bits(cache.layers[l].v, v.data(), r * d) &&
                        same_bits(cache.layers[l].origin, o.data(), r);
        if (!ok) first_bad_layer = static_cast<int>(l);
        cache_equal = ok;
        rows += r;
    }
    std::vector<uint64_t> rpg(rc ? qvref_cache_groups(rc) : 0);
    if (rc) qvref_cache_retained_per_group(rc, rpg.data());
    bool stats_equal = rc && rpg.size() == cache.retained_per_group.size() &&
                       cache.tokens_seen == qvref_cache_tokens_seen(rc) &&
                       cache.peak_group_tokens == qvref_cache_peak_group_tokens(rc) &&
                       cache.value_bytes() == qvref_cache_value_bytes(rc);
    for (size_t i = 0; stats_equal && i < rpg.size(); ++i) stats_equal = rpg[i] == cache.retained_per_group[i];
    std::printf(
        "{\"tokens_equal\": %s, \"query_equal\": %s, \"cache_equal\": %s, \"stats_equal\": %s, \"groups\": %zu, "
        "\"rows\": %zu, \"first_bad_layer\": %d, \"value_bytes\": %llu, \"dropin_ms\": %.3f, "
        "\"reference_ms\": %.3f}\n",
        tokens_equal ? "true" : "false", query_equal ? "true" : "false", cache_equal ? "true" : "false",
        stats_equal ? "true" : "false", groups.size(), rows, first_bad_layer,
        static_cast<unsigned long long>(cache.value_bytes()), dropin_ms, ref_ms);
    if (rc) qvref_cache_destroy(rc);
    qvref_model_destroy(ref);
    return tokens_equal && query_equal && cache_equal && stats_equal ? 0 : 1;
}

std::string catch_msg(const std::function<void()>& f) {
    try {
        f();
    } catch (const qv::Error& e) {
        return e.what();
    }
    return "<no error>";
}

std::string ref_msg(int rc) { return rc == 0 ? "<no error>" : qvref_last_error(); }

void report(const char* name, const std::string& ours, const std::string& ref, bool& all) {
    const bool ok = ours == ref;
    all = all && ok;
    std::printf("%s\t%s\t%s\t%s\n", ok ? "OK" : "MISMATCH", name, ours.c_str(), ref.c_str());
}

int errors() {
    bool all = true;
    std::vector<float> k(8, 1.f), v(8, 1.f), kout(8), vout(8), q(3, 1.f);
    std::vector<uint32_t> idx(8);
    std::vector<double> s(8);
    size_t kept;
    auto prune = [](int scorer, double rho) {
        qv::PruneConfig p;
        p.scorer = static_cast<qv::Scorer>(scorer);
        p.rho = rho;
        return p;
    };
    report("rho_zero", catch_msg([&] { qv::prune_group(k, v, 4, 1, 2, prune(0, 0.0)); }),
           ref_msg(qvref_prune_group(k.data(), 8, v.data(), 8, 4, 1, 2, 0, 0.0, nullptr, 0, kout.data(), vout.data(),
                                     idx.data(), &kept)), all);
    report("rho_gt_one", catch_msg([&] { qv::prune_group(k, v, 4, 1, 2, prune(0, 1.5)); }),
           ref_msg(qvref_prune_group(k.data(), 8, v.data(), 8, 4, 1, 2, 0, 1.5, nullptr, 0, kout.data(), vout.data(),
                                     idx.data(), &kept)), all);
    report("empty_group", catch_msg([&] { qv::prune_group(k, v, 0, 1, 2, prune(0, 0.5)); }),
           ref_msg(qvref_prune_group(k.data(), 8, v.data(), 8, 0, 1, 2, 0, 0.5, nullptr, 0, kout.data(), vout.data(),
                                     idx.data(), &kept)), all);
    report("shape_mismatch", catch_msg([&] { qv::prune_group(k, v, 3, 1, 2, prune(0, 0.5)); }),
           ref_msg(qvref_prune_group(k.data(), 8, v.data(), 8, 3, 1, 2, 0, 0.5, nullptr, 0, kout.data(), vout.data(),
                                     idx.data(), &kept)), all);
    report("identity_skips_shape_check", catch_msg([&] { qv::prune_group(k, v, 3, 1, 2, prune(0, 1.0)); }),
           ref_msg(qvref_prune_group(k.data(), 8, v.data(), 8, 3, 1, 2, 0, 1.0, nullptr, 0, kout.data(), vout.data(),
                                     idx.data(), &kept)), all);
    report("attention_without_query", catch_msg([&] { qv::score_tokens(k, v, 4, 1, 2, qv::Scorer::attention_score); }),
           ref_msg(qvref_score_tokens(k.data(), 8, v.data(), 8, 4, 1, 2, 2, nullptr, 0, s.data())), all);
    report("query_shape", catch_msg([&] { qv::score_tokens(k, v, 4, 1, 2, qv::Scorer::attention_score, q); }),
           ref_msg(qvref_score_tokens(k.data(), 8, v.data(), 8, 4, 1, 2, 2, q.data(), 3, s.data())), all);
    uint64_t gc;
    report("group_count_zero", catch_msg([&] { qv::group_count(10, 0); }), ref_msg(qvref_group_count(10, 0, &gc)),
           all);
    report("unknown_scorer", catch_msg([&] { qv::scorer_from_name("bogus"); }), "unknown scorer: bogus", all);
    qv::ModelConfig bad;
    bad.d_model = 10;
    report("bad_model", catch_msg([&] { qv::StandInModel m(bad); }), "model config: d_model must equal n_h * d_h",
           all);
    report("no_groups", catch_msg([&] {
               qv::ModelConfig c;
               qv::StandInModel m(c);
               qv::prefill(m, {}, qv::PruneConfig{});
           }),
           "prefill: no token groups", all);
    report("empty_frames", catch_msg([&] {
               qv::ModelConfig c;
               qv::StandInModel m(c);
               m.tokenize(qv::FrameBuffer(), 1);
           }),
           "tokenize: empty frame buffer", all);
    report("bad_patch_grid", catch_msg([&] {
               qv::ModelConfig c;
               c.tokens_per_frame = 4;
               qv::StandInModel m(c);
               m.tokenize(qv::FrameBuffer(2, 3, 3), 1);
           }),
           "tokenize: frame size not divisible into the patch grid", all);
    report("project_layer", catch_msg([&] {
               qv::ModelConfig c;
               qv::StandInModel m(c);
               std::vector<float> a, b;
               m.project(qv::TokenGroup{}, 5, a, b);
           }),
           "project: layer out of range", all);
    return all ? 0 : 1;
}

}  // namespace

// Drop-in throughput only (no reference run: at the 7B shape the reference needs ~30 ms per token per layer):
// same arguments as `pipeline`; tokenize + prefill once to warm up (device weights, allocations), then timed `reps`
// times.  Prints {"tokens", "dropin_ms", "tokens_per_s", "rows"}.
int bench(char** a, int reps) {
    const int pattern = std::stoi(a[0]);
    const uint64_t seed = std::stoull(a[1]);
    const size_t frames = std::stoull(a[2]);
    const uint32_t w = std::stoul(a[3]), h = std::stoul(a[4]);
    qv::ModelConfig cfg;
    cfg.d_model = std::stoul(a[5]);
    cfg.n_h = std::stoul(a[6]);
    cfg.d_h = std::stoul(a[7]);
    cfg.layers = std::stoul(a[8]);
    cfg.tokens_per_frame = std::stoul(a[9]);
    cfg.text_tokens = std::stoul(a[10]);
    cfg.seed = seed;
    const uint32_t fpg = std::stoul(a[11]);
    qv::PruneConfig prune;
    prune.scorer = qv::scorer_from_name(a[12]);
    prune.rho = std::stod(a[13]);
    qv::FrameBuffer fb(frames, w, h);
    std::vector<uint8_t> pixels(frames * fb.slot_bytes());
    for (size_t f = 0; f < frames; ++f) {
        qvref_fill_pattern(pattern, seed, f, w, h, pixels.data() + f * fb.slot_bytes());
        fb.write_slot(f, {pixels.data() + f * fb.slot_bytes(), fb.slot_bytes()});
    }
    qv::StandInModel model(cfg);
    size_t rows = 0;
    {
        const auto groups = model.tokenize(fb, fpg);
        rows = qv::prefill(model, groups, prune).retained_tokens();
    }
    double best = 1e30;
    for (int r = 0; r < reps; ++r) {
        const auto t0 = std::chrono::steady_clock::now();
        const auto groups = model.tokenize(fb, fpg);
        const qv::KvCache cache = qv::prefill(model, groups, prune);
        best = std::min(best, std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
    const size_t tokens = frames * cfg.tokens_per_frame;
    std::printf("{\"tokens\": %zu, \"rows\": %zu, \"dropin_ms\": %.3f, \"tokens_per_s\": %.1f}\n", tokens, rows, best,
                tokens / (best / 1e3));
    return 0;
}

// The overlap pipeline (qvx::run_pipeline, include/qv_pipeline.hpp) on a synthetic QVS video encoded by the
// reference: its frame buffer must equal the reference decoder's, its cache the UNMODIFIED reference's prefill of
// those frames (bit for bit); prints the PipelineReport (predicted vs measured t_total) and the sequential
// decode-then-prefill time of the same drop-in calls.
// args: pattern seed frames w h d_model n_h d_h layers tpf text fpg scorer rho cores intervals keyframe_period gap
//       check (0: skip the reference prefill — minutes per 1k tokens at the 7B shape)
int overlap(char** a) {
    const int pattern = std::stoi(a[0]);
    const uint64_t seed = std::stoull(a[1]);
    const size_t frames = std::stoull(a[2]);
    const uint32_t w = std::stoul(a[3]), h = std::stoul(a[4]);
    qv::ModelConfig cfg;
    cfg.d_model = std::stoul(a[5]);
    cfg.n_h = std::stoul(a[6]);
    cfg.d_h = std::stoul(a[7]);
    cfg.layers = std::stoul(a[8]);
    cfg.tokens_per_frame = std::stoul(a[9]);
    cfg.text_tokens = std::stoul(a[10]);
    cfg.seed = seed;
    qvx::PipelineConfig pc;
    pc.frames_per_group = std::stoul(a[11]);
    pc.prune.scorer = qv::scorer_from_name(a[12]);
    pc.prune.rho = std::stod(a[13]);
    pc.cores = std::stoul(a[14]);
    pc.intervals = std::stoul(a[15]);
    qv::EncodeConfig ec;
    ec.keyframe_period = std::stoul(a[16]);
    const uint64_t gap = std::stoull(a[17]);
    const bool check = std::stoi(a[18]) != 0;
    const qv::VideoFile file = qv::synth_video(static_cast<qv::Pattern>(pattern), seed, frames, w, h, ec);
    qv::SampleSpec spec;
    spec.indices = qv::sample_indices_gap(frames, gap);
    qv::StandInModel model(cfg);
    {  // warm-up: device weights, allocations, kernels loaded
        qv::FrameBuffer warm(std::min<size_t>(spec.indices.size(), pc.frames_per_group), w, h);
        qv::prefill(model, model.tokenize(warm, pc.frames_per_group), pc.prune);
    }
    qvx::PipelineReport rep;
    qv::FrameBuffer fb;
    const qv::KvCache cache = qvx::run_pipeline(file, spec, model, pc, &rep, &fb);

    // the sequential composition with the same calls: decode everything, then tokenize + prefill
    const auto s0 = std::chrono::steady_clock::now();
    qv::IntervalSet plan = qv::keyframe_intervals(file, pc.intervals ? pc.intervals : 4 * pc.cores);
    qv::DecodeResult dec = qv::decode_intervals(file, spec, plan, pc.cores);
    const auto s1 = std::chrono::steady_clock::now();
    const qv::KvCache seq = qv::prefill(model, model.tokenize(dec.buffer, pc.frames_per_group), pc.prune);
    const auto s2 = std::chrono::steady_clock::now();
    const bool frames_equal = fb.same_pixels(dec.buffer);

    void* ref = check ? qvref_model_create(cfg.d_model, cfg.n_h, cfg.d_h, cfg.layers, cfg.tokens_per_frame,
                                           cfg.text_tokens, seed)
                      : nullptr;
    void* rc = check ? qvref_prefill_frames(ref, dec.buffer.bytes().data(), dec.buffer.slots(), w, h,
                                            pc.frames_per_group, static_cast<int>(pc.prune.scorer), pc.prune.rho)
                     : nullptr;
    // without the reference: the pipeline's cache must still equal the sequential drop-in composition
    bool cache_equal = cache.layers == seq.layers && (!check || (rc && qvref_cache_layers(rc) == cache.layers.size()));
    for (size_t l = 0; check && cache_equal && l < cache.layers.size(); ++l) {
        const size_t r = qvref_cache_rows(rc, l), d = cfg.d_model;
        std::vector<float> k(r * d), v(r * d);
        std::vector<uint64_t> o(r);
        qvref_cache_copy_layer(rc, l, k.data(), v.data(), o.data());
        cache_equal = same_bits(cache.layers[l].k, k.data(), r * d) && same_bits(cache.layers[l].v, v.data(), r * d) &&
                      same_bits(cache.layers[l].origin, o.data(), r);
    }
    const bool stats_equal = (!check || (rc && cache.tokens_seen == qvref_cache_tokens_seen(rc))) &&
                             cache.tokens_seen == seq.tokens_seen && cache.retained_per_group == seq.retained_per_group;
    const double ms_dec = std::chrono::duration<double, std::milli>(s1 - s0).count();
    const double ms_pre = std::chrono::duration<double, std::milli>(s2 - s1).count();
    std::printf(
        "{\"frames_equal\": %s, \"cache_equal\": %s, \"stats_equal\": %s, \"slots\": %zu, \"groups\": %zu, "
        "\"intervals\": %zu, \"cores\": %zu, \"t_dec_ms\": %.3f, \"t_prefill_ms\": %.3f, \"t_g_dec_ms\": %.3f, "
        "\"t_g_prefill_ms\": %.3f, \"delta_ms\": %.3f, \"t_total_measured_ms\": %.3f, "
        "\"t_total_predicted_ms\": %.3f, \"sequential_decode_ms\": %.3f, \"sequential_prefill_ms\": %.3f, "
        "\"sequential_total_ms\": %.3f}\n",
        frames_equal ? "true" : "false", cache_equal ? "true" : "false", stats_equal ? "true" : "false",
        spec.indices.size(), rep.groups.size(), rep.intervals, pc.cores, rep.t_dec, rep.t_prefill, rep.t_g_dec,
        rep.t_g_prefill, rep.delta, rep.t_total_measured, rep.t_total_predicted, ms_dec, ms_pre, ms_dec + ms_pre);
    if (rc) qvref_cache_destroy(rc);
    if (ref) qvref_model_destroy(ref);
    return frames_equal && cache_equal && stats_equal ? 0 : 1;
}

int main(int argc, char** argv) {
    try {
        if (argc >= 2 && std::string(argv[1]) == "pipeline" && argc == 16) return pipeline(argv + 2);
        if (argc >= 2 && std::string(argv[1]) == "errors") return errors();
        if (argc >= 2 && std::string(argv[1]) == "bench" && argc == 16) return bench(argv + 2, 3);
        if (argc >= 2 && std::string(argv[1]) == "overlap" && argc == 21) return overlap(argv + 2);
    } catch (const std::exception& e) {
        std::printf("{\"exception\": \"%s\"}\n", e.what());
        return 2;
    }
    std::fprintf(stderr, "usage: parity_driver pipeline <14 args> | bench <14 args> | overlap <19 args> | errors\n");
    return 64;
}
