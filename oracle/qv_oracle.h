/* TEST INFRASTRUCTURE ONLY — the CPU restatement used as the parity checker.
 *
 * Plain-C restatement of the QuickPrefill hot path of /root/reference/proj/src/prefill.cpp, plus the pieces the
 * reference does not contain (per-group causal GQA attention, SnapKV observation-window scores, per-head pruning,
 * the group scheduler's offsets).  Every function cites the reference file:line (or PAPER.md line) it follows.
 *
 * Parity pinning: score / retained_count / top_k / gather / tokenize / project / weights are pinned
 * bit-for-bit against the compiled reference (oracle/_ref/libqvref.so) by tests/test_oracle.py.  Attention and
 * SnapKV have no reference implementation: "parity unpinned" — they follow PAPER.md:221-240 and the SnapKV
 * definition stated in DESIGN.md §3.3 and are checked against torch fp64 in tests/test_oracle.py instead.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may call this library.
 */
#ifndef QV_ORACLE_H
#define QV_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* synthetic.cpp:5-10 */
uint64_t qvo_splitmix64(uint64_t* state);
/* prefill.cpp:13-18 */
uint64_t qvo_stream_seed(uint64_t seed, uint32_t tag, uint32_t layer);
/* prefill.cpp:21-30: float((2u-1)*scale), u = (splitmix64>>11)*2^-53 */
void qvo_seeded_matrix(uint64_t seed, uint32_t tag, uint32_t layer, size_t count, double scale, float* out);

/* Synthetic bf16 activations for the device-resident benchmark path: element i of stream
 * (seed, tag, layer, group) is an Irwin-Hall(4) approximate N(0,1) built from splitmix64 output i, scaled by a
 * per-(row, head) factor 2^(j/4), j in [-4, 4] (only when head_scale != 0), rounded RNE to bf16.  Integer-exact, so
 * host and device produce identical bits.  rows x heads x width elements, row-major. */
void qvo_synth_bf16(uint64_t seed, uint32_t tag, uint32_t layer, uint64_t group, size_t rows, uint32_t heads,
                    uint32_t width, int head_scale, uint16_t* out);
float qvo_bf16_to_f32(uint16_t b);
uint16_t qvo_f32_to_bf16(float f);

/* prefill.cpp:200-212 generalised to `heads` independent rows of `width` (per-token mode: heads=1,
 * width=n_h*d_h).  x is (n, heads, width); out is (heads, n): out[h*n+i] = -+sqrt(sum_j double(x)^2),
 * summed sequentially j = 0..width-1 exactly as prefill.cpp:207. negate=1 for key_norm_small. */
void qvo_score_norm(const float* x, size_t n, uint32_t heads, uint32_t width, int negate, double* out);

/* prefill.cpp:213-230: out[i] = (sum_t sum_j double(k[i,j]) * q[t,j]) / (T * n_h), t-outer/j-inner. */
void qvo_score_attention(const float* k, size_t n, uint32_t n_h, uint32_t d_h, const float* q, size_t text_count,
                         double* out);

/* prefill.cpp:235-238 */
size_t qvo_retained_count(double rho, size_t n);

/* prefill.cpp:240-253 restated as a full sort under (score desc, index asc), then ascending indices.
 * Returns the number written (min(k, n)). */
size_t qvo_top_k(const double* scores, size_t n, size_t k, uint32_t* out);

/* prefill.cpp:255-282 per head: for head h, indices = top_k(scores[h*n..], k) and rows gathered.
 * x (n, heads, width) -> out (k, heads, width); idx (k, heads). */
void qvo_gather_heads(const float* x, size_t n, uint32_t heads, uint32_t width, const uint32_t* idx, size_t k,
                      float* out);
size_t qvo_select_heads(const double* scores, size_t n, uint32_t heads, size_t k, uint32_t* idx);

/* Causal GQA attention within one group (no reference code): q (n, n_q, d), k/v (n, n_kv, d),
 * q head h reads kv head h / (n_q / n_kv); o[i,h,:] = sum_{j<=i} softmax_j(scale * q_i.k_j) v_j.  double. */
void qvo_attention(const float* q, const float* k, const float* v, size_t n, uint32_t n_q, uint32_t n_kv,
                   uint32_t d, double scale, double* o);

/* Same as qvo_attention but only for query rows i = row_begin, row_begin + row_step, ... < n (a bounded, unbiased
 * sample for the CPU baseline); o is (n, n_q, d) and only those rows are written.  Returns the rows computed. */
size_t qvo_attention_rows(const float* q, const float* k, const float* v, size_t n, uint32_t n_q, uint32_t n_kv,
                          uint32_t d, double scale, size_t row_begin, size_t row_step, double* o);

/* SnapKV observation-window scores (no reference code): window rows r in [n-W, n), W=min(w,n);
 * s[h, j] = sum_{q heads of kv head h} sum_r softmax_{j<=r}(scale * q_r.k_j)[j]; then optional 1-D average
 * pooling of width `pool` (odd, zero padded, divided by pool).  out is (n_kv, n) double. */
void qvo_snapkv_scores(const float* q, const float* k, size_t n, uint32_t n_q, uint32_t n_kv, uint32_t d,
                       uint32_t window, uint32_t pool, double scale, double* out);

/* Group scheduler (prefill.cpp:170-183, 235-238, 325-328): G = ceil(F / fpg); group g covers frame slots
 * [g*fpg, min((g+1)*fpg, F)), tok_off[g] = g*fpg*tpf; keep[g] = retained_count(rho, N_g); row_off = exclusive
 * prefix sum of keep.  Arrays sized G+1 (tok_off, row_off) and G (keep).  Returns G, or 0 if fpg == 0. */
uint64_t qvo_plan_groups(uint64_t frames, uint32_t fpg, uint32_t tpf, double rho, int64_t* tok_off, int64_t* keep,
                         int64_t* row_off);

#ifdef __cplusplus
}
#endif
#endif
