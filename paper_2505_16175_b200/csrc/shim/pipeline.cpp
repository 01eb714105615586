// The overlap pipeline (SPEC.md:462-535 `overlap_pipeline`) over the drop-in prefill:
// include/qv_pipeline.hpp.
//
// Producer: cfg.cores threads claim the s keyframe intervals earliest first (the claim loop of decode_intervals,
// decode.cpp:196-217) and decode each with the reference's own per-interval worker (decode.cpp:148-174) into a frame
// buffer this pipeline owns — the public decode_intervals keeps its buffer private until every interval is done,
// which is exactly what the overlap must avoid.  Consumer (the calling thread): group g (frame slots
// [g*fpg, min((g+1)*fpg, F)), prefill.cpp:170-183) becomes ready once every interval whose pts range can hold one
// of its frames has finished (and every one of its slots has been written); it is then tokenized and prefilled on
// the GPU through the drop-in's exact kernels — tokenize_group + prefill_group with the tokens kept in HBM,
// bit-identical to the reference — strictly in group order (the cache's append order, prefill.hpp:132-133), while the CPU keeps decoding later intervals.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <exception>
#include <mutex>
#include <thread>

#include "qv_pipeline.hpp"

namespace qv::detail {
// decode.cpp:148-151 (external linkage in the reference's decode.cpp; not declared in its headers).
void decode_one_interval(const VideoFile& file, const ScanResult& scan, const OffsetMap& offsets,
                         uint64_t interval_start, uint64_t interval_end, bool last_interval, FrameBuffer& out,
                         const IntervalHooks* hooks, size_t index);
}  // namespace qv::detail

namespace qv::internal {
// prefill_shim.cpp: tokenize the frames on the device and prefill them as one group (tokens stay in HBM).
void prefill_frames_group(const StandInModel& model, const FrameBuffer& frames, size_t frame_begin, size_t frame_end,
                          const PruneConfig& prune, KvCache& cache);
}  // namespace qv::internal

namespace qvx {
namespace {

using Clock = std::chrono::steady_clock;

double ms(Clock::time_point a, Clock::time_point b) {
    return std::chrono::duration<double, std::milli>(b - a).count();
}

}  // namespace

double predict_latency(double t_dec, double t_prefill, double t_g_dec, double t_g_prefill, double delta) {
    if (t_dec < 0 || t_prefill < 0 || t_g_dec < 0 || t_g_prefill < 0 || delta < 0)
        throw qv::Error("predict_latency: negative input");
    return std::max(t_dec + t_g_prefill, t_prefill + t_g_dec) + delta;
}

qv::KvCache run_pipeline(const qv::VideoFile& file, const qv::SampleSpec& spec, const qv::StandInModel& model,
                         const PipelineConfig& cfg, PipelineReport* report, qv::FrameBuffer* frames_out) {
    const auto t0 = Clock::now();
    spec.validate(file.frame_count);                                       // decode.cpp:181
    if (cfg.cores == 0) throw qv::Error("decode: cores must be >= 1");      // decode.cpp:182
    const size_t slots = spec.indices.size();
    if (slots == 0) throw qv::Error("tokenize: empty frame buffer");                       // prefill.cpp:172
    if (cfg.frames_per_group == 0) throw qv::Error("tokenize: frames_per_group must be >= 1");  // prefill.cpp:173
    const auto [gr, gc] = qv::StandInModel::patch_grid(model.config().tokens_per_frame);
    if (file.height % gr != 0 || file.width % gc != 0)
        throw qv::Error("tokenize: frame size not divisible into the patch grid");
    cfg.prune.validate();  // prefill.cpp:319, after tokenize's checks as in decode -> tokenize -> prefill
    const size_t s = cfg.intervals ? cfg.intervals : 4 * cfg.cores;
    if (s < cfg.cores) throw qv::Error("pipeline: intervals must be >= cores");

    const qv::ScanResult scan = qv::scan_packets(file);
    const qv::IntervalSet plan = qv::keyframe_intervals(scan, s);
    const size_t n = plan.interval_count();
    if (n == 0) throw qv::Error("decode: empty interval plan");             // decode.cpp:183
    const qv::OffsetMap offsets = qv::make_offset_map(spec);
    qv::FrameBuffer buffer(slots, file.width, file.height);

    // Intervals that may write each group's slots: frame f has pts_for_index(f) (exact for the encoder's uniform
    // pts, decode.cpp:76-82); the window is padded by one frame on both sides, so an off-by-one estimate only
    // makes a group wait for one more interval.  A group whose slots are still unwritten after that waits for all.
    const uint32_t fpg = cfg.frames_per_group;
    const size_t G = (slots + fpg - 1) / fpg;
    const uint64_t m = file.frame_count, pad = std::max<uint64_t>(1, file.ticks_per_frame);
    auto interval_of = [&](uint64_t pts) {  // last interval whose start <= pts
        const auto it = std::upper_bound(plan.boundaries.begin(), plan.boundaries.end(), pts);
        const size_t i = it == plan.boundaries.begin() ? 0 : size_t(it - plan.boundaries.begin()) - 1;
        return std::min(i, n - 1);
    };
    std::vector<std::pair<size_t, size_t>> need(G, {n, 0});  // [lo, hi] interval range per group
    for (size_t j = 0; j < slots; ++j) {
        const uint64_t p = m < 2 ? scan.pts_min : qv::pts_for_index(spec.indices[j], scan.pts_min, scan.pts_max, m);
        auto& r = need[j / fpg];
        r.first = std::min(r.first, interval_of(p > pad ? p - pad : 0));
        r.second = std::max(r.second, interval_of(p + pad));
    }

    std::mutex mu;
    std::condition_variable cv;
    std::vector<char> done(n, 0);
    size_t n_done = 0;
    std::exception_ptr error;
    std::atomic<size_t> next{0};
    std::atomic<bool> failed{false};
    Clock::time_point first_start = Clock::time_point::max(), last_done = t0;
    auto worker = [&] {
        for (;;) {
            if (failed.load(std::memory_order_relaxed)) break;
            const size_t i = next.fetch_add(1, std::memory_order_relaxed);  // earliest first
            if (i >= n) break;
            const auto ts = Clock::now();
            {
                std::lock_guard<std::mutex> lk(mu);
                first_start = std::min(first_start, ts);
            }
            try {
                const auto [a, b] = plan.interval(i);
                qv::detail::decode_one_interval(file, scan, offsets, a, b, plan.is_last(i), buffer, nullptr, i);
            } catch (...) {
                std::lock_guard<std::mutex> lk(mu);
                if (!error) error = std::current_exception();
                failed.store(true, std::memory_order_relaxed);
            }
            {
                std::lock_guard<std::mutex> lk(mu);
                done[i] = 1;
                ++n_done;
                last_done = Clock::now();
            }
            cv.notify_all();
        }
        std::lock_guard<std::mutex> lk(mu);
        cv.notify_all();
    };
    std::vector<std::thread> pool;
    const size_t workers = std::min(cfg.cores, n);
    pool.reserve(workers);
    for (size_t w = 0; w < workers; ++w) pool.emplace_back(worker);

    qv::KvCache cache = qv::make_cache(model.config());
    if (cfg.prune.rho > 0.0 && cfg.prune.rho <= 1.0) {  // the cache's final size is static (prefill.cpp:304-308 appends retained_count rows per group): reserve it
        // once, so appending group by group never reallocates and copies the rows already there
        size_t rows = 0;
        for (size_t g = 0; g < G; ++g) {
            const size_t f0 = g * fpg, f1 = std::min<size_t>(f0 + fpg, slots);
            rows += qv::retained_count(cfg.prune.rho, (f1 - f0) * model.config().tokens_per_frame);
        }
        for (qv::LayerCache& l : cache.layers) {
            l.k.reserve(rows * model.config().d_model);
            l.v.reserve(rows * model.config().d_model);
            l.origin.reserve(rows);
        }
    }
    std::vector<GroupTiming> times(G);
    double t_prefill = 0, t_last = 0;
    try {
        for (size_t g = 0; g < G; ++g) {
            const size_t f0 = g * fpg, f1 = std::min<size_t>(f0 + fpg, slots);
            {
                std::unique_lock<std::mutex> lk(mu);
                cv.wait(lk, [&] {
                    if (error || n_done == n) return true;
                    for (size_t i = need[g].first; i <= need[g].second; ++i)
                        if (!done[i]) return false;
                    for (size_t j = f0; j < f1; ++j)
                        if (buffer.fill_count(j) == 0) return false;
                    return true;
                });
                if (error) break;
            }
            times[g].ready_ms = ms(t0, Clock::now());
            const auto a = Clock::now();
            qv::internal::prefill_frames_group(model, buffer, f0, f1, cfg.prune, cache);
            const auto b = Clock::now();
            times[g].start_ms = ms(t0, a);
            times[g].done_ms = ms(t0, b);
            t_last = ms(a, b);
            t_prefill += t_last;
        }
    } catch (...) {
        failed.store(true, std::memory_order_relaxed);
        for (auto& t : pool) t.join();
        throw;
    }
    for (auto& t : pool) t.join();
    if (error) std::rethrow_exception(error);
    const auto t_end = Clock::now();

    if (report) {
        PipelineReport& r = *report;
        r.intervals = n;
        r.delta = ms(t0, first_start);
        r.t_dec = ms(first_start, last_done);
        r.t_g_dec = std::max(0.0, times[0].ready_ms - r.delta);
        r.t_prefill = t_prefill;
        r.t_g_prefill = t_last;
        r.t_total_measured = ms(t0, t_end);
        r.t_total_predicted = predict_latency(r.t_dec, r.t_prefill, r.t_g_dec, r.t_g_prefill, r.delta);
        r.groups = std::move(times);
    }
    if (frames_out) *frames_out = std::move(buffer);
    return cache;
}

}  // namespace qvx
