// qv_pipeline.hpp — the overlap pipeline of the paper (§3.3; SPEC.md:462-535 `overlap_pipeline`)
// over the drop-in prefill: CPU decoding of s >> c keyframe intervals, earliest first, feeds group-wise GPU prefill as
// soon as each group's frames are in the frame buffer.  Not part of the reference's headers (the reference specifies
// the module but never implemented it); it builds on the reference's unchanged video side (decode.hpp, interval.hpp:
// the producer is the reference's own per-interval worker) and on the drop-in qv:: prefill (libqv_prefill.so), and
// lives in libqv_pipeline.so.
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

#include "qv/decode.hpp"
#include "qv/prefill.hpp"

namespace qvx {

/// SPEC.md PipelineConfig: s = intervals (s >= c >= 1), c = decode cores.
struct PipelineConfig {
    size_t intervals = 0;            // s; 0 = 4 * cores (SPEC.md design decision)
    size_t cores = 1;                // c
    uint32_t frames_per_group = 16;
    qv::PruneConfig prune;
};

struct GroupTiming {
    double ready_ms = 0;   // every frame of the group decoded (from pipeline start)
    double start_ms = 0;   // prefill of the group started
    double done_ms = 0;    // its pruned rows are in the cache
};

/// SPEC.md PipelineReport.  Stage times in ms: t_dec / t_g_dec from the first interval's start, Δ = start of the
/// pipeline -> first interval start (metadata scan, interval plan, setup).
struct PipelineReport {
    double t_dec = 0, t_prefill = 0, t_g_dec = 0, t_g_prefill = 0, delta = 0;
    double t_total_measured = 0, t_total_predicted = 0;
    size_t intervals = 0;
    std::vector<GroupTiming> groups;
};

/// t_total = max(t_dec + t^g_prefill, t_prefill + t^g_dec) + Δ.  Throws qv::Error on a negative input.
double predict_latency(double t_dec, double t_prefill, double t_g_dec, double t_g_prefill, double delta);

/// Decode `spec`'s frames of `file` with cfg.cores workers over cfg.intervals keyframe intervals (earliest first,
/// decode.cpp:196-217) and prefill group g on the GPU as soon as its frames are decoded, strictly in group order
/// (prefill.hpp:132-133).  The cache — and `frames_out`, when given — are bit-identical to
/// decode_intervals(...) -> model.tokenize(buffer, fpg) -> qv::prefill(model, groups, prune).
qv::KvCache run_pipeline(const qv::VideoFile& file, const qv::SampleSpec& spec, const qv::StandInModel& model,
                         const PipelineConfig& cfg, PipelineReport* report = nullptr,
                         qv::FrameBuffer* frames_out = nullptr);

}  // namespace qvx
