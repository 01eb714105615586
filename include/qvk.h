/* qvk.h — C ABI of the B200-native (sm_100a) QuickPrefill hot path.
 *
 * The reference (/root/reference/proj) exposes QuickPrefill only as the C++ API of include/qv/prefill.hpp
 * (std::span / std::vector / exceptions, no C ABI).  This header is the thin C layer underneath it:
 *   - paper_2505_16175_b200/csrc/shim/prefill_shim.cpp implements the UNCHANGED qv:: API of prefill.hpp on top
 *     of these entry points (that shim is the drop-in for src/prefill.cpp — see INTEGRATION.md);
 *   - Python (ctypes) and C callers use them directly for the batched, device-resident path.
 *
 * Conventions
 *   - Plain pointers and sizes only.  "_d" pointers are device (HBM) pointers, others are host pointers.
 *   - Device entry points are asynchronous and stream-ordered on `stream` (a cudaStream_t; NULL = legacy
 *     default stream).  They never synchronise unless documented.
 *   - Return 0 on success.  QVK_E_INVALID (-1) carries the reference's qv::Error text verbatim (the shim throws
 *     qv::Error(qvk_last_error())); QVK_E_CUDA (-2) a CUDA runtime failure; QVK_E_UNSUPPORTED (-3) a shape this
 *     build has no kernel for.  qvk_last_error() is thread-local.
 *   - Groups (prefill.hpp:27-35 TokenGroup) are described by qvk_groups: group g owns token rows
 *     [tok_off[g], tok_off[g+1]) of the q/k/v tensors and cache rows [row_off[g], row_off[g]+keep[g]).
 *   - K/V/Q rows are (tokens, heads, width) row-major ("NHD", prefill.hpp:49-51).  Scores are (group, head, token):
 *     scores[heads*tok_off[g] + h*N_g + i].  Selected indices and the cache are (cache row, head):
 *     idx[(row_off[g]+r)*heads + h], k_cache[((row_off[g]+r)*heads + h)*width + c], origin likewise.
 *     Per-token pruning (the reference's unchanged semantics, prefill.hpp:105-108) is heads = 1, width = n_h*d_h.
 */
#ifndef QVK_H
#define QVK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* qvk_stream_t; /* == cudaStream_t */

enum {
    QVK_OK = 0,
    QVK_E_INVALID = -1,
    QVK_E_CUDA = -2,
    QVK_E_UNSUPPORTED = -3,
};

enum { QVK_F32 = 0, QVK_BF16 = 1 };

/* Values 0..2 equal qv::Scorer (prefill.hpp:37); 3 is the SnapKV observation-window scorer (north star (3)). */
enum { QVK_KEY_NORM_SMALL = 0, QVK_VALUE_NORM = 1, QVK_ATTENTION_SCORE = 2, QVK_SNAPKV = 3 };

typedef struct {
    int32_t n_groups;            /* G >= 1 */
    int64_t max_tokens;          /* max_g N_g (launch sizing) */
    int64_t total_tokens;        /* tok_off[G] (rows of q/k/v) */
    int64_t total_rows;          /* row_off[G] (sum of keep) */
    const int64_t* tok_off_d;    /* [G+1] token row offsets into q/k/v */
    const int64_t* keep_d;       /* [G]   retained tokens per group (= retained_count(rho, N_g)) */
    const int64_t* row_off_d;    /* [G+1] cache row offsets (exclusive prefix sum of keep) */
    const uint64_t* first_token_d; /* [G] global token id of the group's row 0 (prefill.hpp:29) */
} qvk_groups;

const char* qvk_last_error(void);
int qvk_version(void);
int qvk_device_count(int* out);

/* ---- device memory / stream plumbing (so C++ callers such as the shim need no CUDA headers) ---------------- */
int qvk_malloc(void** out_d, size_t bytes);
int qvk_free(void* p_d);
int qvk_memcpy_h2d(void* dst_d, const void* src, size_t bytes, qvk_stream_t stream);
int qvk_memcpy_d2h(void* dst, const void* src_d, size_t bytes, qvk_stream_t stream);
int qvk_stream_sync(qvk_stream_t stream);
/* Synchronous copies between PAGEABLE host memory (e.g. the std::vectors of the reference's API) and the device,
 * ordered after the work already on `stream`: staged through pinned double buffers, the DMA of one chunk overlapping
 * the multi-threaded host copy of the previous one (plain cudaMemcpy from pageable memory runs at ~2 GB/s D2H on the
 * B200 box, the staged copy at several times that). */
int qvk_memcpy_d2h_pageable(void* dst, const void* src_d, size_t bytes, qvk_stream_t stream);
int qvk_memcpy_h2d_pageable(void* dst_d, const void* src, size_t bytes, qvk_stream_t stream);

/* ---- (a1) group scheduler, host side ------------------------------------------------------------------------- */
/* prefill.cpp:325-328 group_count; "frames_per_group must be >= 1" on fpg == 0. */
int qvk_group_count(uint64_t total_frames, uint32_t frames_per_group, uint64_t* out);
/* prefill.cpp:235-238 retained_count: min(n, max(1, llround(rho*n))). */
size_t qvk_retained_count(double rho, size_t token_count);
/* prefill.cpp:65-67 PruneConfig::validate: "retention ratio must be in (0, 1]". */
int qvk_validate_rho(double rho);
/* Plans G = ceil(F/fpg) groups of tpf tokens per frame (prefill.cpp:170-183, last group short), retained counts
 * and cache offsets, and a contiguous partition of the groups over `world` ranks balanced by attention cost
 * (sum N_g^2): rank r owns groups [rank_begin[r], rank_begin[r+1]).  Arrays: tok_off/row_off G+1, keep G,
 * rank_begin world+1 (may be NULL when world <= 1).  Call with tok_off == NULL to get G only (in *n_groups). */
int qvk_plan_groups(uint64_t total_frames, uint32_t frames_per_group, uint32_t tokens_per_frame, double rho,
                    int32_t world, uint64_t* n_groups, int64_t* tok_off, int64_t* keep, int64_t* row_off,
                    int32_t* rank_begin);

/* ---- (a5)/(a6)/(a7) importance scores --------------------------------------------------------------------------- */
/* key_norm_small / value_norm (prefill.cpp:200-212): per (token, head) -+sqrt(sum_j double(x_j)^2) summed
 * sequentially over j = 0..width-1 in double — bit-identical to the reference.  attention_score
 * (prefill.cpp:213-230, heads must be 1): (sum_t sum_j double(k_j)*q_tj)/(T*n_h) in the reference's order,
 * bit-identical; `n_h` is only the divisor.  Shape errors carry the reference's messages. */
int qvk_score(qvk_stream_t stream, const qvk_groups* groups, const void* k_d, const void* v_d, int dtype,
              int32_t heads, int32_t width, int32_t scorer, const float* text_query_d, int64_t text_count,
              int32_t n_h, double* scores_d);

/* GQA attention_score (prefill.cpp:213-230 generalised to n_q query / n_kv KV heads):
 *   qbar[h, j] = (float) sum_t sum_{hq in group(h)} double(text_query[t, hq, j])   (t outer, hq inner)
 *   per_head = 1: s[i, h] = (sum_{j < d_h} double(k[i, h, j]) * qbar[h, j]) / (T * n_q / n_kv)
 *   per_head = 0: s[i]    = (sum_{j < n_kv d_h} double(k[i, :, :]) * qbar[:, :]) / (T * n_q)
 * i.e. the reference's own attention_score applied to the ONE pre-summed text-query row qbar (sum over j in the
 * reference's sequential double order, bit-identical to qv::score_tokens(k, v, N, n_h, d_h, attention_score, qbar)
 * up to the divisor), an HBM-bound GEMV instead of the reference's O(N*T*D) loop.  text_query_d (text_count, n_q,
 * d_h) fp32; k_d (tokens, n_kv, d_h) bf16; qbar_ws_d receives qbar (n_kv * d_h floats; may be NULL = scratch);
 * scores in the qvk_score layout (heads = per_head ? n_kv : 1).  Errors: "attention_score scorer requires a text
 * query" when text_count == 0. */
int qvk_text_query_sum(qvk_stream_t stream, const float* text_query_d, int64_t text_count, int32_t n_q, int32_t n_kv,
                       int32_t d_h, float* qbar_d);
int qvk_score_text(qvk_stream_t stream, const qvk_groups* groups, const void* k_d, int32_t n_q, int32_t n_kv,
                   int32_t d_h, int32_t per_head, const float* text_query_d, int64_t text_count, float* qbar_ws_d,
                   double* scores_d);

/* SnapKV observation-window scores per KV head: window = the last min(window, N_g) tokens of
 * the group; s[h, j] = sum over the n_q/n_kv query heads of h and the window rows r of causal
 * softmax_j(scale * q_r . k_j); optional average pooling of odd width `pool` (1 = none).  bf16 q/k, fp32 math,
 * scores written as double in the qvk_score layout (heads = n_kv). */
int qvk_snapkv_score(qvk_stream_t stream, const qvk_groups* groups, const void* q_d, const void* k_d,
                     int32_t n_q, int32_t n_kv, int32_t d_h, int32_t window, int32_t pool, float scale,
                     double* scores_d);
/* The same scores given the window rows' softmax statistics (qvk_attention_window_stats), so only the second pass
 * (per-key sums of the normalised probabilities) runs.  d_h == 128.  qvk_prefill_layer does this itself when it
 * prunes with SnapKV: the layer's attention kernel writes the statistics. */
int qvk_snapkv_score_stats(qvk_stream_t stream, const qvk_groups* groups, const void* q_d, const void* k_d,
                           int32_t n_q, int32_t n_kv, int32_t d_h, int32_t window, int32_t pool, float scale,
                           const float* window_stats_d, double* scores_d);

/* ---- (a9) top-k selection -------------------------------------------------------------------------------------- */
/* Per (group, head): the keep[g] best scores under (score desc, index asc), -0.0 == +0.0, written ascending
 * (prefill.cpp:240-253) to idx_d[(row_off[g]+r)*heads + h].  Exact radix select on the 64-bit keys. */
int qvk_select(qvk_stream_t stream, const qvk_groups* groups, const double* scores_d, int32_t heads,
               uint32_t* idx_d);

/* ---- (a10)/(a11) KV compaction into the cache ------------------------------------------------------------------- */
/* k_cache[(row_off[g]+r), h, :] = k[tok_off[g] + idx[...], h, :] (same for v); origin = first_token[g] + idx
 * (prefill.cpp:277-280, 304-308).  idx_d == NULL means the rho == 1 identity (prefill.cpp:263-270): every row kept
 * in order (requires keep[g] == N_g).  origin_d may be NULL. */
int qvk_gather(qvk_stream_t stream, const qvk_groups* groups, const void* k_d, const void* v_d, int dtype,
               int32_t heads, int32_t width, const uint32_t* idx_d, void* k_cache_d, void* v_cache_d,
               uint64_t* origin_d);

/* score -> select -> gather (prune_group for every group of the batch).  scores_ws_d must hold
 * heads * tok_off[G] doubles and idx_ws_d total_rows * heads uint32 (either may be NULL: then the call allocates
 * and frees stream-ordered scratch).  rho == 1 takes the identity path without scoring (prefill.cpp:263-270). */
int qvk_prune(qvk_stream_t stream, const qvk_groups* groups, const void* k_d, const void* v_d, int dtype,
              int32_t heads, int32_t width, int32_t scorer, double rho, const float* text_query_d,
              int64_t text_count, int32_t n_h, double* scores_ws_d, uint32_t* idx_ws_d, void* k_cache_d,
              void* v_cache_d, uint64_t* origin_d);

/* select -> gather from precomputed scores (any scorer, e.g. qvk_snapkv_score's), one cluster launch per batch
 * (prune_fused.cu): bf16 rows of 64/128/256/512 elements, groups of at most 65536 tokens; other shapes run the
 * separate qvk_select + qvk_gather kernels.  Same outputs as qvk_select followed by qvk_gather; idx_d may be NULL. */
int qvk_select_gather(qvk_stream_t stream, const qvk_groups* groups, const double* scores_d, const void* k_d,
                      const void* v_d, int dtype, int32_t heads, int32_t width, uint32_t* idx_d, void* k_cache_d,
                      void* v_cache_d, uint64_t* origin_d);

/* ---- (a4) per-group causal GQA attention ------------------------------------------------------------------------ */
/* O[i, h, :] = sum_{j <= i, same group} softmax_j(scale * Q[i,h].K[j,h/(n_q/n_kv)]) V[j, ...]; bf16 in/out, fp32
 * accumulate.  tcgen05/TMEM/TMA kernel; d_h == 64 or 128 (QVK_E_UNSUPPORTED otherwise). */
int qvk_attention(qvk_stream_t stream, const qvk_groups* groups, const void* q_d, const void* k_d,
                  const void* v_d, int32_t n_q, int32_t n_kv, int32_t d_h, float scale, void* o_d);
/* qvk_attention that also writes the softmax statistics of every group's last `window` query rows (SnapKV's
 * observation window): window_stats_d[(g * n_q + h) * window + r] = m + log2(l) of query row N_g - window + r, head
 * h, in the scaled log2 domain (m = the row's running max of scale * log2(e) * q.k, l = sum_j 2^(that - m));
 * rows before the group start are not written.  d_h == 128. */
int qvk_attention_window_stats(qvk_stream_t stream, const qvk_groups* groups, const void* q_d, const void* k_d,
                               const void* v_d, int32_t n_q, int32_t n_kv, int32_t d_h, float scale, void* o_d,
                               int32_t window, float* window_stats_d);

/* ---- one full pruned-prefill layer for all groups of the batch -------------------------------------------------- */
typedef struct {
    int32_t n_q, n_kv, d_h;   /* GQA shape; K/V rows are (tokens, n_kv, d_h) */
    int32_t scorer;           /* QVK_KEY_NORM_SMALL / QVK_VALUE_NORM / QVK_ATTENTION_SCORE / QVK_SNAPKV */
    int32_t per_head;         /* 1: prune each KV head independently (north star (4)); 0: per token (reference) */
    double rho;               /* retention ratio (0, 1] */
    float scale;              /* softmax scale, usually 1/sqrt(d_h) */
    int32_t snap_window, snap_pool;
    /* QVK_ATTENTION_SCORE only: the text-token queries (text_count, n_q, d_h) fp32 on the device — the reference's
     * StandInModel::text_query() (prefill.cpp:108-113) in GQA form; scored through qvk_score_text. */
    const float* text_query_d;
    int64_t text_count;
} qvk_layer_params;

/* attention -> score -> select -> gather for one layer.  scores_ws_d: n_kv * tok_off[G] doubles; idx_ws_d:
 * total_rows * n_kv uint32 (NULL -> stream-ordered scratch).  With rho == 1 (identity, prefill.cpp:263-270) idx_ws_d
 * receives 0..keep-1 per group like every scored path. */
int qvk_prefill_layer(qvk_stream_t stream, const qvk_groups* groups, const qvk_layer_params* p, const void* q_d,
                      const void* k_d, const void* v_d, void* o_d, double* scores_ws_d, uint32_t* idx_ws_d,
                      void* k_cache_d, void* v_cache_d, uint64_t* origin_d);

/* ---- per-model / per-video context: the plan on the device and every workspace, allocated once -------------------- */
/* The reference builds its StandInModel once and shares it read-only (prefill.hpp:72); a serving loop over the layers
 * of a video (and over consecutive videos of the same shape) should likewise pay allocation, plan upload and
 * workspace sizing once.  qvk_ctx_create takes the group plan on the HOST (tok_off: n_groups + 1 token offsets,
 * first_token: n_groups global token ids, NULL = tok_off) and the layer parameters; it computes keep / row_off
 * (retained_count, prefill.cpp:235-238), uploads them, and allocates the scores / idx / text-query workspaces on the
 * current device.  qvk_ctx_groups returns the device descriptor (valid until qvk_ctx_destroy) for the other entry
 * points; qvk_ctx_prefill_layer(_x) run one layer with the context's plan, parameters and workspaces (no allocation,
 * no host synchronisation).  A context may be used from one stream at a time. */
typedef struct qvk_ctx_st* qvk_ctx_t;
int qvk_ctx_create(qvk_ctx_t* out, const qvk_layer_params* p, int32_t n_groups, const int64_t* tok_off,
                   const uint64_t* first_token);
int qvk_ctx_groups(qvk_ctx_t ctx, qvk_groups* out);
int qvk_ctx_prefill_layer(qvk_ctx_t ctx, qvk_stream_t stream, const void* q_d, const void* k_d, const void* v_d,
                          void* o_d, void* k_cache_d, void* v_cache_d, uint64_t* origin_d);
int qvk_ctx_prefill_layer_x(qvk_ctx_t ctx, qvk_stream_t stream, const void* x_d, int32_t d_model, const void* w_d,
                            void* q_ws_d, void* k_ws_d, void* v_ws_d, void* o_d, void* k_cache_d, void* v_cache_d,
                            uint64_t* origin_d);
int qvk_ctx_destroy(qvk_ctx_t ctx);

/* ---- §8f-1: QKV projection (tcgen05 GEMM) with the key-norm score fused into its epilogue ------------------------ */
/* [Q | K | V] = X . W^T: x_d (tokens, d_model) bf16, w_d ((n_q + 2 n_kv) d_h, d_model) bf16 row-major (the
 * nn.Linear layout of the stacked q/k/v projection weights); outputs q_d (tokens, n_q, d_h), k_d / v_d
 * (tokens, n_kv, d_h) bf16, fp32 accumulation.  The stand-in of the reference is prefill.cpp:185-190 (K, V only).
 * When scores_d is not NULL the epilogue also writes the key_norm_small score of every (token, KV head) of the
 * stored bf16 K (prefill.cpp:200-212 order, bit-identical to qvk_score with heads = n_kv, width = d_h) in the
 * qvk_score layout of `groups` (which must cover the tokens).  Needs d_model % 64 == 0, 256 % d_h == 0 and
 * (n_q + 2 n_kv) d_h % 256 == 0 (QVK_E_UNSUPPORTED otherwise). */
int qvk_project_qkv(qvk_stream_t stream, const void* x_d, int64_t tokens, int32_t d_model, const void* w_d,
                    int32_t n_q, int32_t n_kv, int32_t d_h, void* q_d, void* k_d, void* v_d,
                    const qvk_groups* groups, double* scores_d);

/* One pruned-prefill layer from hidden states: qvk_project_qkv (key-norm fused when p->scorer is key_norm_small and
 * p->per_head) -> attention -> select + gather into the cache (other scorers: their score kernel first).
 * q_ws_d / k_ws_d / v_ws_d receive the projections; scores_ws_d: n_kv * tokens doubles (required). */
int qvk_prefill_layer_x(qvk_stream_t stream, const qvk_groups* groups, const qvk_layer_params* p, const void* x_d,
                        int32_t d_model, const void* w_d, void* q_ws_d, void* k_ws_d, void* v_ws_d, void* o_d,
                        double* scores_ws_d, uint32_t* idx_ws_d, void* k_cache_d, void* v_cache_d,
                        uint64_t* origin_d);

/* ---- multi-GPU: the cache all-gather fused into the compaction (peer memory over NVLink) ----------------------- */
/* CUDA IPC export / import of a device buffer (e.g. a rank's cache) so other ranks can store into it directly:
 * handle_out receives 64 bytes, offset_out the buffer's offset inside its allocation.  qvk_ipc_open maps the
 * allocation of another process (base_out) — the buffer is base_out + offset; qvk_ipc_close unmaps it. */
int qvk_ipc_get_handle(const void* ptr_d, void* handle_out, uint64_t* offset_out);
int qvk_ipc_open(const void* handle, void** base_out);
int qvk_ipc_close(void* base_d);
/* qvk_prune / qvk_prefill_layer whose compaction stores every retained row into n_dest caches (<= 8): dest 0 is this
 * GPU's cache, the others the same cache buffers of the other ranks (qvk_ipc_open pointers), so after every rank's
 * call (and a cross-rank barrier) each GPU holds the whole pruned cache — no separate all-gather.  kc_d / vc_d /
 * origin_d are HOST arrays of n_dest device pointers (origin_d may be NULL).  bf16 rows of 64/128/256/512 with the
 * key_norm_small / value_norm scorers (QVK_E_UNSUPPORTED otherwise). */
int qvk_prune_dests(qvk_stream_t stream, const qvk_groups* groups, const void* k_d, const void* v_d, int32_t heads,
                    int32_t width, int32_t scorer, double rho, double* scores_ws_d, uint32_t* idx_ws_d, int32_t n_dest,
                    void* const* kc_d, void* const* vc_d, uint64_t* const* origin_d);
/* Device-side barrier after a *_dests call (no host synchronisation): every rank adds 1 to every rank's 32-bit
 * counter (flags_d: HOST array of the n ranks' counter addresses, own included — qvk_ipc_open mappings; zeroed once)
 * and waits on the device until its own counter reaches epoch * n (epoch = 1, 2, ... per call); later work on
 * `stream` then sees every peer's stores.  A rank that does not arrive within QVK_PEER_BARRIER_TIMEOUT_MS (20 s)
 * sets *err_d to 1 instead of hanging. */
int qvk_peer_barrier(qvk_stream_t stream, int32_t n, uint32_t* const* flags_d, int32_t self, uint32_t epoch,
                     uint32_t* err_d);
int qvk_prefill_layer_dests(qvk_stream_t stream, const qvk_groups* groups, const qvk_layer_params* p, const void* q_d,
                            const void* k_d, const void* v_d, void* o_d, double* scores_ws_d, uint32_t* idx_ws_d,
                            int32_t n_dest, void* const* kc_d, void* const* vc_d, uint64_t* const* origin_d);

/* ---- multi-GPU: the cache all-gather as ONE NCCL collective call over NVLink / NVSwitch ------------------------ */
/* Groups are independent and every cache offset is a pure function of (rho, N_g), so rank r writes its
 * groups' pruned rows at their global offsets (qvk_plan_groups rank_begin) and one collective replicates the cache
 * for the decode step — the reference's single-writer, in-order KvCache (prefill.hpp:132-133) assembled on every
 * GPU.  NCCL has no all-gather-v, so qvk_allgather_layer issues one in-place ncclBroadcast per source rank and
 * buffer inside ONE ncclGroupStart/End (a single fused NCCL launch); rank_row_begin (host, world + 1 entries) gives
 * the first cache row of each rank's segment (row_off[rank_begin[r]]).  k/v caches hold heads * width bf16 per
 * row, origin heads uint64 per row (may be NULL).  Stream-ordered on `stream`.
 *   qvk_comm_unique_id   rank 0 creates the 128-byte ncclUniqueId; the caller ships it to the other ranks
 *   qvk_comm_init        one rank per process on the current device (ncclCommInitRankConfig); for world > 1 NCCL
 *                        is capped at QVK_COMM_CTAS CTAs (default 8, world 1: 0; 0 = NCCL's choice) and as many SMs are
 *                        reserved (qvk_reserve_sms) until qvk_comm_destroy, so the persistent kernels never wait
 *                        for SMs held by an all-gather overlapping them
 *   qvk_comm_init_all    one process driving n_dev GPUs (ncclCommInitAll): comms_out[i] drives devices[i]; wrap
 *                        the per-device calls in qvk_comm_group_start / qvk_comm_group_end
 *   qvk_comm_wrap        adopt a caller's ncclComm_t (not destroyed by qvk_comm_destroy)
 *   qvk_comm_check       ncclCommGetAsyncError: QVK_E_CUDA with NCCL's message after an asynchronous failure */
typedef struct qvk_comm_st* qvk_comm_t;
int qvk_comm_unique_id(void* id_out);
int qvk_comm_init(qvk_comm_t* out, int32_t world, int32_t rank, const void* unique_id);
int qvk_comm_init_all(qvk_comm_t* comms_out, int32_t n_dev, const int32_t* devices);
int qvk_comm_wrap(qvk_comm_t* out, void* nccl_comm);
int qvk_comm_rank(qvk_comm_t comm, int32_t* rank, int32_t* world);
int qvk_comm_check(qvk_comm_t comm);
int qvk_comm_destroy(qvk_comm_t comm);
int qvk_comm_group_start(void);
int qvk_comm_group_end(void);
int qvk_allgather_layer(qvk_stream_t stream, qvk_comm_t comm, const int64_t* rank_row_begin, int32_t heads,
                        int32_t width, void* k_cache_d, void* v_cache_d, uint64_t* origin_d);
/* SMs the persistent kernels (attention, projection: one CTA per SM walking a static work list) leave free for
 * kernels running beside them on other streams — a collective, a decoder.  Their grids become SM count - n (>= 2).
 * Results do not depend on it.  0 <= n < SM count; returns the previous value in *previous (may be NULL). */
int qvk_reserve_sms(int32_t n, int32_t* previous);

/* ---- diagnostics ------------------------------------------------------------------------------------------------ */
/* Route the last qvk_prune / qvk_prefill_layer* call of this thread took for its prune step: 0 = fused cluster
 * kernel (score + select + gather in one launch), 1 = separate score / select / gather kernels, 2 = rho == 1
 * identity copy, 3 = select + gather on precomputed scores (fused), -1 = none yet. */
int qvk_last_prune_route(void);

/* ---- §8f-4: decode-step consumer of the pruned cache ------------------------------------------------------------- */
/* O[t, h] = softmax_r(scale * q[t, h] . K[r, h / (n_q/n_kv)]) V[r, ...] over every cache row r (non-causal: the video
 * tokens precede the queries) and lse[t, h] = ln sum_r exp(scale * q . K[r]) (may be NULL) so the caller can merge it
 * with its own text-token attention.  q_d / o_d (n_tq, n_q, d_h) bf16; k_cache_d / v_cache_d (rows, n_kv, d_h) bf16 —
 * one layer of the per-head pruned cache (qvk_prefill_layer's layout).  d_h == 128.  Split-KV: ws_d must hold
 * qvk_decode_workspace(...) bytes. */
int qvk_decode_workspace(int32_t n_tq, int32_t n_q, int32_t n_kv, int32_t d_h, int64_t rows, size_t* bytes);
int qvk_decode_attention(qvk_stream_t stream, const void* q_d, int32_t n_tq, int32_t n_q, int32_t n_kv, int32_t d_h,
                         const void* k_cache_d, const void* v_cache_d, int64_t rows, float scale, void* o_d,
                         float* lse_d, void* ws_d, size_t ws_bytes);

/* ---- stand-in model pieces of the reference API (exact, for the drop-in shim) ----------------------------------- */
/* prefill.cpp:21-30 seeded_matrix generated on the device, bit-identical (counter-based splitmix64). */
int qvk_seeded_matrix(qvk_stream_t stream, uint64_t seed, uint32_t tag, uint32_t layer, size_t count, double scale,
                      float* out_d);
/* prefill.cpp:38-54 matmul: out(rows, d_out) = x(rows, d_in) * w(d_in, d_out), double accumulation in the
 * reference's sequential order (no FMA) — bit-identical fp32 output. */
int qvk_project_exact(qvk_stream_t stream, const float* x_d, int64_t rows, int32_t d_in, const float* w_d,
                      int32_t d_out, float* out_d);
/* prefill.cpp:123-168 tokenize_group body: frames are (n_frames, 3, height, width) uint8 slots; tokens
 * (n_frames * tpf, d_model) fp32; embed (d_model, 3).  Bit-identical.  "tokenize: frame size not divisible into
 * the patch grid" on a bad size. */
int qvk_tokenize(qvk_stream_t stream, const uint8_t* frames_d, int64_t n_frames, uint32_t width, uint32_t height,
                 uint32_t tokens_per_frame, const float* embed_d, int32_t d_model, float* tokens_d);
/* Same tokens rounded to bf16 (RNE): the activations X of qvk_project_qkv (video frames -> pruned cache). */
int qvk_tokenize_bf16(qvk_stream_t stream, const uint8_t* frames_d, int64_t n_frames, uint32_t width, uint32_t height,
                      uint32_t tokens_per_frame, const float* embed_d, int32_t d_model, void* tokens_d);
/* prefill.cpp:116-121 */
void qvk_patch_grid(uint32_t tokens_per_frame, uint32_t* rows, uint32_t* cols);

/* ---- synthetic device-resident inputs (benchmark / tests; same bits as oracle qvo_synth_bf16) ------------------- */
int qvk_synth_bf16(qvk_stream_t stream, uint64_t seed, uint32_t tag, uint32_t layer, uint64_t group, int64_t rows,
                   int32_t heads, int32_t width, int32_t head_scale, void* out_d);

#ifdef __cplusplus
}
#endif
#endif /* QVK_H */
