// (a4) Per-group causal GQA attention prefill on sm_100a: TMA -> smem ring -> tcgen05.mma into TMEM, online
// softmax in registers, P kept in TMEM (TS-MMA), no reference counterpart.
//
// Persistent kernel: one CTA per SM loops over work units in heaviest-first order (unit = group g, query head hq,
// query-tile pair p: two 128-row query tiles, rows [256p, 256p+256) of the group, sharing every K/V tile the CTA
// streams; the second tile needs one extra, diagonal, K/V tile).  Consecutive units of a CTA overlap: the next
// unit's Q load and first S MMAs run while the dedicated epilogue warpgroup drains the previous unit's O.
//
// Warp roles (512 threads):
//   warps 0-3   softmax for query tile 0   (thread = one TMEM lane = one query row; the whole S row is thread-local)
//   warps 4-7   softmax for query tile 1
//   warps 8-11  epilogue: O / l -> bf16 -> HBM, then release O's TMEM columns to the MMA warp
//   warp  12    TMA producer  (Q0, Q1 per unit; K0, V0, K1, V1, ... through a 4-stage 32 KB ring)
//   warp  13    MMA issuer    (one elected lane) + TMEM owner (512 columns: S0 | S1 | O0 | O1, 128 each)
// MMA order per K/V step j (FA4-style ping-pong, so the tensor pipe works on one tile while the other's softmax
// runs):  PV0(j)  S0(j+1)  PV1(j)  S1(j+1).  P_t(j) (bf16) is written by the softmax warps over the first 64 columns
// of S_t and consumed as the TMEM A operand of PV_t(j); tcgen05 ops execute in issue order, so S_t(j+1) (issued
// after PV_t(j)) never overwrites P_t(j) early, and the commit of S_t(j+1) also proves PV_t(j) retired — which is
// what lets the softmax warps rescale O_t in TMEM (lazily, only when a row max grows by > 2^8) without another
// barrier.  PV_t(0) of a unit (accumulate = 0) waits until the epilogue released O_t of the previous unit.
//
// Layouts: Q/K/V are (tokens, heads, 128) bf16.  Each 128x128 tile lands in smem as two 128-row x 128-byte
// SWIZZLE_128B chunks (d 0..63, d 64..127) via 3-D TMA boxes {64, 1, 128}.  S = Q K^T uses K-major A and B
// descriptors (SBO 1024 B); O += P V uses V as an MN-major B operand (LBO 16 KB between the d chunks, SBO 1024 B).
// Algorithmic FLOPs per (group, q head): 4 * d * N (N + 1) / 2 (causal, diagonal included; masked work uncredited).
#include <cudaTypedefs.h>

#include <cstdlib>

#include "common.cuh"
#include "ptx.cuh"

namespace qvk {
namespace {

constexpr int kBM = 128;                      // query rows per tile
constexpr int kBN = 128;                      // kv rows per tile
constexpr int kStages = 3;                    // K/V ring depth
constexpr int kQBufs = 2;                     // Q double buffer: the next unit's Q loads during the current one
constexpr uint32_t kChunkBytes = kBM * 64 * 2; // one 128-row x 128-byte SW128 chunk (64 head-dim columns)
// Head dim D in {64, 128}: a 128-row Q/K/V tile is D/64 chunks.
template <int D>
__host__ __device__ constexpr uint32_t tile_bytes() { return kChunkBytes * (D / 64); }
constexpr int kThreads = 512;                 // 4 warpgroups: softmax0, softmax1, epilogue, {TMA, MMA, 2 spare}
constexpr int kEpiWarp0 = 8;
constexpr int kTmaWarp = 12;
constexpr int kMmaWarp = 13;
// Launch pool 512 * 128 registers: 2*128*184 (softmax) + 128*48 (epilogue) + 128*96 (TMA/MMA) = 65536.
constexpr int kRegsSoftmax = 184;
constexpr int kRegsEpilogue = 48;
constexpr int kRegsProducer = 96;
constexpr float kRescaleThreshold = 8.0f;     // log2 units: rescale O only when a row max grows by > 256x

#ifdef QVK_ATTN_TRACE
// Debug timeline (tools/attn_trace.cu): clock64 stamps of CTA 0's first (heaviest) unit.  With
// QVK_ATTN_TRACE_UNITS=4 the first four units of CTA 0 are traced instead (units of <= 8 K/V steps, e.g. 1024-token
// groups): unit u's stamps are shifted by 64 slots inside the MMA (0..255) and per-tile softmax (512 + 256 t) areas.
__device__ long long g_attn_trace[1024];
#ifndef QVK_ATTN_TRACE_UNITS
#define QVK_ATTN_TRACE_UNITS 1
#endif
#define QVK_TRACE(slot)                                                                   \
    do {                                                                                  \
        if (blockIdx.x == 0 && unit_iter < QVK_ATTN_TRACE_UNITS) {                        \
            long long _c;                                                                 \
            asm volatile("mov.u64 %0, %%clock64;" : "=l"(_c));                            \
            const int _s = (slot);                                                        \
            g_attn_trace[_s >= 1000 ? _s : _s + unit_iter * 64] = _c;                     \
        }                                                                                 \
    } while (0)
#else
#define QVK_TRACE(slot) \
    do {                \
    } while (0)
#endif

#ifdef QVK_ATTN_UNITLOG
// Debug per-unit log (tools/attn_unitlog.cu): the MMA thread of every CTA stamps clock64 at the top of each of its
// first 128 valid units (and once after the last), with the unit's K/V step count.
__device__ long long g_attn_unitlog[1024][129][3];
#define QVK_ULOG(i, nkv)                                                                  \
    do {                                                                                  \
        if (blockIdx.x < 1024 && (i) < 129) {                                             \
            long long _g;                                                                 \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_g));                        \
            g_attn_unitlog[blockIdx.x][(i)][0] = clock64();                               \
            g_attn_unitlog[blockIdx.x][(i)][1] = (nkv);                                   \
            g_attn_unitlog[blockIdx.x][(i)][2] = _g;                                      \
        }                                                                                 \
    } while (0)
#else
#define QVK_ULOG(i, nkv) \
    do {                 \
    } while (0)
#endif

#ifdef QVK_ATTN_STALLS
// Debug stall accounting (tools/attn_stalls.cu): clock64 cycles per CTA spent in each barrier wait category.
//   0 MMA: q_full  1 MMA: kv_full  2 MMA: o_free  3 MMA: p_full  4 MMA: loop total  5 units (MMA)
//   6 softmax tile 0 (warp 0 lane 0): s_full   7 epilogue (warp 8 lane 0): l_full + o_done
__device__ unsigned long long g_attn_stall[1024][8];
#define QVK_SWAIT(cat, b, ph)                                                                  \
    do {                                                                                       \
        const long long _s0 = clock64();                                                       \
        ptx::mbar_wait((b), (ph));                                                             \
        if (blockIdx.x < 1024) g_attn_stall[blockIdx.x][(cat)] += clock64() - _s0;             \
    } while (0)
#define QVK_SWAIT_T(tid, cat, b, ph)                                                           \
    do {                                                                                       \
        const long long _s0 = clock64();                                                       \
        ptx::mbar_wait((b), (ph));                                                             \
        if (threadIdx.x == (tid) && blockIdx.x < 1024) g_attn_stall[blockIdx.x][(cat)] += clock64() - _s0; \
    } while (0)
#define QVK_STALL_ADD(cat, v) \
    do {                      \
        if (blockIdx.x < 1024) g_attn_stall[blockIdx.x][(cat)] += (v); \
    } while (0)
#else
#define QVK_SWAIT(cat, b, ph) ptx::mbar_wait((b), (ph))
#define QVK_SWAIT_T(tid, cat, b, ph) ptx::mbar_wait((b), (ph))
#define QVK_STALL_ADD(cat, v) \
    do {                      \
    } while (0)
#endif

struct AttnParams {
    const int64_t* tok_off;
    int n_groups;
    int n_q;
    int n_kv;
    int tiles_max;
    int total_units;
    float scale_log2;
    __nv_bfloat16* o;
    int pre_issue;  // issue the next unit's S0(0) during tile 1's lone last step (QVK_ATTN_PRE=0 disables)
    int gblock;     // groups per block of the unit order (= n_groups: one block)
    float* lse;     // optional: softmax statistics m + log2(l) (scaled log2 domain) of each group's last lse_window
    int lse_window; // query rows, [group][query head][window row] — SnapKV's pass 1 (snapkv.cu) for free
};

struct Barriers {
    uint64_t q_full[kQBufs];
    uint64_t q_empty[kQBufs];
    uint64_t kv_full[kStages];
    uint64_t kv_empty[kStages];
    uint64_t s_full[2];
    uint64_t p_full[2][2];  // [tile][half]: P columns 0..63 / 64..127 of the tile are in TMEM
    uint64_t o_done[2];     // last PV of the tile retired (MMA commit)
    uint64_t o_free[2];     // epilogue has O_t in registers: TMEM columns reusable (128 arrivals)
    uint64_t l_full[2];     // softmax published the row sums of the tile (128 arrivals)
    uint64_t l_free[2];     // epilogue has read them (128 arrivals).  Keeps the softmax at most one unit ahead of
                            // the epilogue: with 1-step units nothing else does, and l_full's phase parity would alias
    uint32_t tmem_base;
    float row_sum[2][kBM];  // [tile][row]
};

template <int D>
constexpr size_t smem_bytes() { return (2 * kQBufs + kStages) * tile_bytes<D>() + sizeof(Barriers); }

// Descriptor of the same operand at a byte offset: only the 14-bit start-address field (addr >> 4, bits 0-13)
// changes and it cannot carry (shared memory < 256 KB), so one 32-bit add on the low word — instead of rebuilding
// the descriptor (shift, mask, or, ~4 uniform-datapath ops) for each of the 8 k-steps of every MMA.
__device__ __forceinline__ uint64_t desc_plus(uint64_t d, uint32_t off_bytes) {
    const uint32_t lo = static_cast<uint32_t>(d) + (off_bytes >> 4);
    return (d & 0xffffffff00000000ull) | lo;
}
__device__ __forceinline__ uint32_t kmajor_off(int kk) { return (kk >> 2) * kChunkBytes + (kk & 3) * 32; }
__device__ __forceinline__ uint64_t kmajor_desc(uint32_t tile_addr, int kk) {
    // k-step kk (16 elements) of a K-major SW128 tile: chunk kk/4, +32 B per step inside the 128-byte row.
    return ptx::umma_desc_sw128(tile_addr + (kk >> 2) * kChunkBytes + (kk & 3) * 32, 16, 1024);
}
__device__ __forceinline__ uint64_t mnmajor_desc(uint32_t tile_addr, int kk) {
    // k-step kk (16 kv rows) of the MN-major V tile: +16 rows * 128 B; the two 64-wide d chunks are LBO apart.
    return ptx::umma_desc_sw128(tile_addr + kk * 16 * 128, kChunkBytes, 1024);
}

// Work units, heaviest first: a unit is two 128-row query tiles 2p, 2p+1 of one query head (rows
// [256p, 256p+256) of the group) sharing one K/V stream (tile 2p+1 needs one extra, diagonal, step).  Pairs from the
// last one down, then group, then query head fastest, so the CTAs running concurrently share K/V through L2.
// (Pairing the same tile of two query heads of a KV head — equal step counts — measured 3 % slower on B200.)
struct Unit {
    int g, hk, hq0, hq1, mt0, mt1, n, n0, n1, nkv;
    int64_t tok0;
    bool valid;
};
// The groups are taken in blocks of p.gblock: all units of a block (heaviest pair level first) before the next block,
// so a group's K/V is streamed from DRAM about once instead of once per pair level (with one block for the whole
// launch, a C4 group's K/V was re-read ~8x: 27 GB of DRAM reads per launch for 8.5 GB of Q, K and V).
__device__ __forceinline__ Unit decode_unit(const AttnParams& p, int u) {
    Unit w;
    if (u >= p.total_units) {  // the look-ahead past a CTA's last unit: no loads
        w.valid = false;
        w.g = w.hk = w.hq0 = w.hq1 = w.mt0 = w.mt1 = w.n = w.n0 = w.n1 = w.nkv = 0;
        w.tok0 = 0;
        return w;
    }
    const int pairs = (p.tiles_max + 1) / 2;
    const int per_block = p.gblock * p.n_q * pairs;
    const int blk = u / per_block;
    const int gb = min(p.gblock, p.n_groups - blk * p.gblock);  // groups in this block (the last may be short)
    const int per_pair = gb * p.n_q;
    const int ub = u - blk * per_block;
    const int pair = pairs - 1 - ub / per_pair;
    const int rem = ub % per_pair;
    const int gi = rem / p.n_q;  // group inside the block
    w.g = blk * p.gblock + gi;
    w.hq0 = w.hq1 = rem - gi * p.n_q;
    w.hk = w.hq0 / (p.n_q / p.n_kv);
    w.tok0 = __ldg(p.tok_off + w.g);
    w.n = static_cast<int>(__ldg(p.tok_off + w.g + 1) - w.tok0);
    w.mt0 = 2 * pair;
    w.mt1 = 2 * pair + 1;
    w.valid = w.mt0 * kBM < w.n;
    w.n0 = w.mt0 + 1;                           // K/V tiles of query tile 0 (last one is diagonal)
    w.n1 = w.mt1 * kBM < w.n ? w.mt1 + 1 : 0;   // K/V tiles of query tile 1 (0: tile absent)
    w.nkv = w.n1 ? w.n1 : w.n0;
    return w;
}

template <int D, int kPolyPairs>
__global__ void __launch_bounds__(kThreads, 1)
    attention_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                         const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o,
                         const AttnParams p) {
    constexpr uint32_t kTileBytes = tile_bytes<D>();
    // 228 KB of tiles + barriers leave no room for alignment slack: the dynamic window must be 1024-aligned
    // (SWIZZLE_128B atoms); checked below.
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sQ = smem;                                   // [Q buffer][tile 0 | tile 1]
    uint8_t* sKV = smem + 2 * kQBufs * kTileBytes;        // ring
    Barriers* bar = reinterpret_cast<Barriers*>(smem + (2 * kQBufs + kStages) * kTileBytes);
    if (ptx::smem_u32(smem) & 1023) __trap();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int unit_iter = 0;  // per-role count of valid units processed (barrier phases; trace)
    if (threadIdx.x == 0) QVK_TRACE(1022);
    // PDL: a dependent launched with programmatic stream serialization (the fused prune of qvk_prefill_layer, which
    // does not read O) may be scheduled now; its CTAs take the SMs this persistent grid releases in its tail.
    if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    if (threadIdx.x == 0) {
        for (int b = 0; b < kQBufs; ++b) {
            ptx::mbar_init(&bar->q_full[b], 1);
            ptx::mbar_init(&bar->q_empty[b], 2);  // the unit's last S MMA retired + its O stores have left the buffer
        }
        for (int s = 0; s < kStages; ++s) {
            ptx::mbar_init(&bar->kv_full[s], 1);
            ptx::mbar_init(&bar->kv_empty[s], 1);
        }
        for (int t = 0; t < 2; ++t) {
            ptx::mbar_init(&bar->s_full[t], 1);
            ptx::mbar_init(&bar->p_full[t][0], 128);
            ptx::mbar_init(&bar->p_full[t][1], 128);
            ptx::mbar_init(&bar->o_done[t], 1);
            ptx::mbar_init(&bar->o_free[t], 128);
            ptx::mbar_init(&bar->l_full[t], 128);
            ptx::mbar_init(&bar->l_free[t], 128);
        }
        ptx::fence_mbar_init();
    }
    if (warp == kMmaWarp) ptx::tmem_alloc<512>(&bar->tmem_base);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = bar->tmem_base;

    // Register rebalancing (warpgroup-uniform).
    if (warp >= kTmaWarp) {
        if (kRegsProducer < 128) ptx::setmaxnreg_dec<kRegsProducer>();
        if (warp == kTmaWarp && ptx::elect_one()) {
            // ===================== TMA producer =====================
            ptx::prefetch_tmap(&tm_q);
            ptx::prefetch_tmap(&tm_k);
            ptx::prefetch_tmap(&tm_v);
            // Q of unit i goes to buffer i & 1 and is issued early in unit i-1 (after its first K/V tiles, by
            // which time unit i-2's S MMAs — the previous users of that buffer — have retired).
            auto next_valid = [&](int u) -> int {
                for (; u < p.total_units; u += gridDim.x)
                    if (decode_unit(p, u).valid) return u;
                return p.total_units;
            };
            // Q of unit qi goes to buffer qi & 1 once q_empty says its previous user (unit qi - 2) is done with it.
            // block = false: only if that is already the case (the buffer is also the previous unit's O staging
            // area, released by the epilogue — not worth stalling the K/V stream for).
            auto load_q = [&](const Unit& w, int qi, bool block) -> bool {
                const int qb = qi & 1;
                uint8_t* q_dst = sQ + qb * 2 * kTileBytes;
                const uint32_t ph = ((qi >> 1) & 1) ^ 1;
                if (!block && !ptx::mbar_test(&bar->q_empty[qb], ph)) return false;
                ptx::mbar_wait(&bar->q_empty[qb], ph);
                ptx::mbar_arrive_expect_tx(&bar->q_full[qb], w.n1 ? 2 * kTileBytes : kTileBytes);
                const int r0 = static_cast<int>(w.tok0) + w.mt0 * kBM;
                const int r1 = static_cast<int>(w.tok0) + w.mt1 * kBM;
#pragma unroll
                for (int c = 0; c < D / 64; ++c) {
                    ptx::tma_load_3d(q_dst + c * kChunkBytes, &tm_q, &bar->q_full[qb], 64 * c, w.hq0, r0);
                    if (w.n1)
                        ptx::tma_load_3d(q_dst + kTileBytes + c * kChunkBytes, &tm_q, &bar->q_full[qb], 64 * c, w.hq1,
                                         r1);
                }
                return true;
            };
            uint32_t item = 0;
            int u = next_valid(blockIdx.x);
            if (u < p.total_units) load_q(decode_unit(p, u), 0, true);
            for (; u < p.total_units; ++unit_iter) {
                const Unit w = decode_unit(p, u);
                const int un = next_valid(u + gridDim.x);
                const int q_at = min(2, 2 * w.nkv - 1);  // K/V item from which the next unit's Q may be issued
                bool q_pending = un < p.total_units;
                for (int it = 0; it < 2 * w.nkv; ++it, ++item) {
                    const uint32_t st = item % kStages;
                    ptx::mbar_wait(&bar->kv_empty[st], ((item / kStages) & 1) ^ 1);
                    const CUtensorMap* map = (it & 1) ? &tm_v : &tm_k;
                    const int row = static_cast<int>(w.tok0) + (it >> 1) * kBN;
                    uint8_t* dst = sKV + st * kTileBytes;
                    ptx::mbar_arrive_expect_tx(&bar->kv_full[st], kTileBytes);
#pragma unroll
                    for (int c = 0; c < D / 64; ++c)
                        ptx::tma_load_3d(dst + c * kChunkBytes, map, &bar->kv_full[st], 64 * c, w.hk, row);
                    // non-blocking from q_at on, blocking at the unit's last item (the next unit needs its Q)
                    if (q_pending && it >= q_at)
                        q_pending = !load_q(decode_unit(p, un), unit_iter + 1, it == 2 * w.nkv - 1);
                }
                u = un;
            }
        } else if (warp == kMmaWarp && ptx::elect_one()) {
            // ===================== MMA issuer =====================
            constexpr uint32_t kIdS = ptx::idesc_bf16_f32(kBM, kBN, false, false);
            constexpr uint32_t kIdPV = ptx::idesc_bf16_f32(kBM, D, false, true);
            const uint32_t q_base = ptx::smem_u32(sQ);
            const uint32_t ring = ptx::smem_u32(sKV);
            uint32_t item = 0;
            uint32_t pv_step[2] = {0, 0};  // P publications consumed per tile (p_full phases)
            uint32_t o_units[2] = {0, 0};  // units per tile (o_free phases)
            bool s0_pre = false;           // S0(0) of this unit was issued ahead, during the previous unit's last step
#ifdef QVK_ATTN_STALLS
            const long long loop0 = clock64();
#endif
            auto wait_item = [&](uint32_t it) -> uint32_t {
                const uint32_t st = it % kStages;
                QVK_SWAIT(1, &bar->kv_full[st], (it / kStages) & 1);
                ptx::tc_fence_after();
                return ring + st * kTileBytes;
            };
            // S_t(j) = Q_t K(j)^T into TMEM columns [128 t, 128 t + 128)
            auto issue_s_at = [&](int t, uint32_t qa, uint32_t k_addr) {
                const uint64_t dq = kmajor_desc(qa, 0), dk = kmajor_desc(k_addr, 0);
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk)
                    ptx::mma_ss(tmem + t * 128, desc_plus(dq, kmajor_off(kk)), desc_plus(dk, kmajor_off(kk)), kIdS,
                                kk > 0);
            };
            // The next valid unit is decoded one unit ahead (two L2 loads + four integer divisions, ~1200 cycles of
            // this single thread, tools/attn_trace.cu), and a pre-issued unit skips its Q / K(0) waits (already
            // satisfied at the pre-issue): the unit boundary is on the tensor pipe's critical path.
            auto next_valid = [&](int u) -> int {
                for (; u < p.total_units; u += gridDim.x)
                    if (decode_unit(p, u).valid) return u;
                return p.total_units;
            };
            int u = next_valid(blockIdx.x);
            Unit w = decode_unit(p, u);
            while (u < p.total_units) {
                QVK_TRACE(39);  // unit loop top
                QVK_ULOG(unit_iter, w.nkv);
                QVK_TRACE(23);  // decoded
                const int nt[2] = {w.n0, w.n1};
                const int qb = unit_iter & 1;
                const uint32_t q_addr = q_base + qb * 2 * kTileBytes;
                if (!s0_pre) QVK_SWAIT(0, &bar->q_full[qb], (unit_iter >> 1) & 1);
                QVK_TRACE(31);  // Q ready
                ptx::tc_fence_after();
                auto issue_s = [&](int t, uint32_t k_addr) { issue_s_at(t, q_addr + t * kTileBytes, k_addr); };
                // O_t += P_t(j) V(j), in two halves as the softmax publishes P (p_full[t][0], p_full[t][1]).
                auto issue_pv = [&](int t, uint32_t v_addr, int j) {
                    if (j == 0) QVK_SWAIT(2, &bar->o_free[t], (o_units[t] & 1) ^ 1);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        QVK_SWAIT(3, &bar->p_full[t][h], pv_step[t] & 1);
                        QVK_TRACE(j * 8 + 1 + 3 * t + h);
                        ptx::tc_fence_after();
                        const uint64_t dv = mnmajor_desc(v_addr, 0);
#pragma unroll
                        for (int kk = 4 * h; kk < 4 * h + 4; ++kk)
                            ptx::mma_ts(tmem + 256 + t * 128, tmem + t * 128 + kk * 8, desc_plus(dv, kk * 16 * 128),
                                        kIdPV, (j > 0 || kk > 0) ? 1u : 0u);
                    }
                    ++pv_step[t];
                    if (j == nt[t] - 1) {
                        ptx::mma_commit(&bar->o_done[t]);
                        ++o_units[t];
                    }
                };
                const uint32_t k0 = s0_pre ? ring + (item % kStages) * kTileBytes : wait_item(item);
                QVK_TRACE(15);  // K(0) ready
                if (!s0_pre) {
                    issue_s(0, k0);
                    ptx::mma_commit(&bar->s_full[0]);
                }
                if (w.n1) {
                    issue_s(1, k0);
                    ptx::mma_commit(&bar->s_full[1]);
                }
                QVK_TRACE(7);  // S1(0) issued
                if (w.nkv == 1) ptx::mma_commit(&bar->q_empty[qb]);  // every S of the unit issued
                ptx::mma_commit(&bar->kv_empty[item % kStages]);
                bool next_pre = false;
                const int un = next_valid(u + gridDim.x);  // off the critical path: S0(0) / S1(0) are queued
                const Unit wn = decode_unit(p, un);
                for (int j = 0; j < w.nkv; ++j) {
                    const uint32_t v_item = item + 2 * j + 1;
                    const uint32_t v_addr = wait_item(v_item);
                    QVK_TRACE(j * 8);
                    const bool more = j + 1 < w.nkv;
                    if (j < w.n0) issue_pv(0, v_addr, j);
                    uint32_t kn = 0;
                    if (more) kn = wait_item(v_item + 1);
                    if (j + 1 < w.n0) {
                        issue_s(0, kn);
                        ptx::mma_commit(&bar->s_full[0]);
                        QVK_TRACE(j * 8 + 3);
                    }
                    if (j < w.n1) issue_pv(1, v_addr, j);
                    ptx::mma_commit(&bar->kv_empty[v_item % kStages]);
                    if (j + 1 < w.n1) {
                        issue_s(1, kn);
                        ptx::mma_commit(&bar->s_full[1]);
                        QVK_TRACE(j * 8 + 6);
                    }
                    if (j + 2 == w.nkv) ptx::mma_commit(&bar->q_empty[qb]);  // the unit's last S was just issued
                    if (more) ptx::mma_commit(&bar->kv_empty[(v_item + 1) % kStages]);
                    // Tile 1 has one more (diagonal) step than tile 0: while its softmax runs that last step alone,
                    // start the next unit — its S0(0) goes into tile 0's free S columns (P0's last PV was issued
                    // above), so the next unit's tile-0 softmax overlaps this unit's tail.  K(0) of the next unit
                    // is the ring item after this unit's last V; the two slots released above let it load.
                    if (p.pre_issue && j + 2 == w.nkv && w.n1 == w.n0 + 1) {
                        if (un < p.total_units) {
                            const int qbn = (unit_iter + 1) & 1;
                            QVK_SWAIT(0, &bar->q_full[qbn], ((unit_iter + 1) >> 1) & 1);
                            ptx::tc_fence_after();
                            const uint32_t kn0 = wait_item(item + 2 * w.nkv);
                            issue_s_at(0, q_base + qbn * 2 * kTileBytes, kn0);
                            ptx::mma_commit(&bar->s_full[0]);
                            next_pre = true;
                        }
                    }
                }
                QVK_TRACE((w.nkv - 1) * 8 + 7);  // unit's MMAs all issued
                item += 2 * w.nkv;
                ++unit_iter;
                s0_pre = next_pre;
                QVK_STALL_ADD(5, 1);
                u = un;
                w = wn;
            }
            QVK_ULOG(unit_iter, 0);
#ifdef QVK_ATTN_STALLS
            QVK_STALL_ADD(4, clock64() - loop0);
#endif
        }
    } else if (warp >= kEpiWarp0) {
        ptx::setmaxnreg_dec<kRegsEpilogue>();
        // ===================== epilogue: O / l -> bf16 -> HBM =====================
        // Full 128-row tiles are staged (bf16, SWIZZLE_128B) in the unit's own Q tile buffer — dead once the tile's
        // last S MMA retired, which o_done implies — and written by TMA stores: one thread per row storing its own
        // 256-byte row touched 32 lines per warp instruction and held the LSU for ~2000 cycles per tile, right at the
        // unit boundary where the MMA thread's loads / barrier waits queue behind it (per-unit overhead 3230 -> 1960
        // cycles with the stores removed, tools/attn_unitlog.cu).  Rows past the group's end (its last, partial
        // tile) would overwrite the next group: that tile is stored row by row.  The buffer is handed back to the
        // producer (q_empty, 2nd arrival) once the TMA engine has read it.
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
        const bool leader = warp == kEpiWarp0 && lane == 0;
        if (leader) ptx::prefetch_tmap(&tm_o);
        uint32_t t_units[2] = {0, 0};
        for (int u = blockIdx.x; u < p.total_units; u += gridDim.x) {
            const Unit w = decode_unit(p, u);
            if (!w.valid) continue;
            const int qb = unit_iter & 1;
            for (int t = 0; t < 2; ++t) {
                if (t == 1 && !w.n1) continue;
                const uint32_t ph = t_units[t] & 1;
                QVK_SWAIT_T(256, 7, &bar->l_full[t], ph);
                const float inv = 1.f / bar->row_sum[t][row];
                ptx::mbar_arrive(&bar->l_free[t]);
                QVK_SWAIT_T(256, 7, &bar->o_done[t], ph);
                ptx::tc_fence_after();
                const uint32_t o_col = tmem + lane_off + 256 + t * 128;
                const int mt = t ? w.mt1 : w.mt0;
                const int qrow = mt * kBM + row;
                __nv_bfloat16* dst = p.o + ((w.tok0 + qrow) * p.n_q + (t ? w.hq1 : w.hq0)) * static_cast<int64_t>(D);
                const bool staged = (mt + 1) * kBM <= w.n;  // warp-uniform (whole tile inside the group)
                uint8_t* stage = sQ + qb * 2 * kTileBytes + t * kTileBytes;
#pragma unroll
                for (int c = 0; c < D / 16; ++c) {
                    uint32_t o[16];
                    QVK_TMEM_LD16(o_col + c * 16, o);
                    ptx::tmem_ld_wait();
                    if (c == D / 16 - 1) {  // all of O_t has been read: hand its TMEM columns back to the MMA warp
                        ptx::tc_fence_before();
                        ptx::mbar_arrive(&bar->o_free[t]);
                    }
                    uint32_t pk[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e)
                        pk[e] = ptx::pack_bf16(__uint_as_float(o[2 * e]) * inv, __uint_as_float(o[2 * e + 1]) * inv);
                    if (staged) {
                        // columns 16c..16c+15 = 16-byte units 2(c%4), 2(c%4)+1 of row `row` in d-chunk c/4, XOR-swizzled
                        const uint32_t base = ptx::smem_u32(stage) + (c >> 2) * kChunkBytes + row * 128;
                        const uint32_t u0 = static_cast<uint32_t>(2 * (c & 3));
                        ptx::sts128(base + ((u0 ^ (row & 7)) << 4), pk[0], pk[1], pk[2], pk[3]);
                        ptx::sts128(base + (((u0 + 1) ^ (row & 7)) << 4), pk[4], pk[5], pk[6], pk[7]);
                    } else if (qrow < w.n) {
                        uint4* d4 = reinterpret_cast<uint4*>(dst + c * 16);
                        d4[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                        d4[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
                    }
                }
                if (staged) {
                    ptx::fence_proxy_async_smem();  // generic st.shared -> the TMA engine (async proxy)
                    ptx::named_bar_sync(1, 128);    // the four epilogue warps' rows are all in the stage
                    if (leader) {
#pragma unroll
                        for (int ch = 0; ch < D / 64; ++ch)
                            ptx::tma_store_3d(&tm_o, stage + ch * kChunkBytes, 64 * ch, t ? w.hq1 : w.hq0,
                                              static_cast<int>(w.tok0) + mt * kBM);
                        ptx::bulk_commit_group();
                    }
                }
                ++t_units[t];
            }
            if (leader) {  // the stores of this unit have read the buffer: the producer may load Q into it again
                ptx::bulk_wait_group_read<0>();
                ptx::mbar_arrive(&bar->q_empty[qb]);
            }
            ++unit_iter;
        }
        if (leader) ptx::bulk_wait_group<0>();  // every O store complete before the CTA retires
    } else {
        ptx::setmaxnreg_inc<kRegsSoftmax>();
        // ===================== softmax (+ lazy O correction) =====================
        const int t = warp >> 2;                 // query tile handled by this warpgroup
        const int quarter = warp & 3;            // TMEM lane quarter this warp may access
        const int row = quarter * 32 + lane;
        const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
        const uint32_t s_col = tmem + lane_off + t * 128;
        const uint32_t o_col = tmem + lane_off + 256 + t * 128;
        const float sl2 = p.scale_log2;
        uint32_t step = 0;   // S tiles consumed (s_full phases)
        uint32_t units = 0;  // units with this tile (row_sum buffer / l_full phases)
        for (int u = blockIdx.x; u < p.total_units; u += gridDim.x) {
            const Unit w = decode_unit(p, u);
            if (!w.valid) continue;
            const int mt = t ? w.mt1 : w.mt0;
            const int nt = t ? w.n1 : w.n0;
            if (nt == 0) {
                ++unit_iter;
                continue;
            }
            float m_ref = -INFINITY, l = 0.f;
            for (int j = 0; j < nt; ++j, ++step) {
                QVK_SWAIT_T(0, 6, &bar->s_full[t], step & 1);
                if (row == 0) QVK_TRACE(512 + t * 256 + j * 8);
                ptx::tc_fence_after();
                float x[128];
                QVK_TMEM_LD32F(s_col + 0, (x + 0));
                QVK_TMEM_LD32F(s_col + 32, (x + 32));
                QVK_TMEM_LD32F(s_col + 64, (x + 64));
                QVK_TMEM_LD32F(s_col + 96, (x + 96));
                ptx::tmem_ld_wait();
                if (j == mt) {
#pragma unroll
                    for (int c = 0; c < 128; ++c)
                        if (c > row) x[c] = -INFINITY;
                }
                float mx0 = x[0], mx1 = x[1], mx2 = x[2], mx3 = x[3];
#pragma unroll
                for (int c = 4; c < 128; c += 4) {
                    mx0 = fmaxf(mx0, x[c]);
                    mx1 = fmaxf(mx1, x[c + 1]);
                    mx2 = fmaxf(mx2, x[c + 2]);
                    mx3 = fmaxf(mx3, x[c + 3]);
                }
                const float mx = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3));
                if (row == 0) QVK_TRACE(512 + t * 256 + j * 8 + 1);
                const float m_new = mx * sl2;
                if (j == 0) {
                    m_ref = m_new;
                } else {
                    const bool need = m_new > m_ref + kRescaleThreshold;
                    if (__any_sync(0xffffffffu, need)) {
                        const float m_upd = need ? m_new : m_ref;
                        const float f = ptx::ex2(m_ref - m_upd);
                        l *= f;
                        m_ref = m_upd;
#pragma unroll
                        for (int c = 0; c < D / 16; ++c) {
                            uint32_t o[16];
                            QVK_TMEM_LD16(o_col + c * 16, o);
                            ptx::tmem_ld_wait();
#pragma unroll
                            for (int e = 0; e < 16; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * f);
                            QVK_TMEM_ST16(o_col + c * 16, o);
                        }
                        ptx::tmem_st_wait();
                    }
                }
                const ptx::f2 sl2x2 = ptx::f2_make(sl2, sl2);
                const ptx::f2 negx2 = ptx::f2_make(-m_ref, -m_ref);
                ptx::f2 acc0 = ptx::f2_make(0.f, 0.f), acc1 = acc0;
                // 16 exponential pairs (32 P columns = 16 packed TMEM columns) per part; x*scale - max on FFMA2,
                // 2^x on the MUFU except kPolyPairs of every 16 pairs on the FMA pipe (ex2_poly2).
                auto part = [&](int q, uint32_t (&pk)[16]) {
#pragma unroll
                    for (int c = 0; c < 16; ++c) {
                        const int xc = 32 * q + 2 * c;
                        const ptx::f2 y = ptx::f2_fma(ptx::f2_make(x[xc], x[xc + 1]), sl2x2, negx2);
                        float p0, p1;
                        ptx::f2_split(y, p0, p1);
                        if (c < kPolyPairs) {
                            ptx::ex2_poly2(p0, p1);
                        } else {
                            p0 = ptx::ex2(p0);
                            p1 = ptx::ex2(p1);
                        }
                        if (c & 1) acc1 = ptx::f2_add(acc1, ptx::f2_make(p0, p1));
                        else acc0 = ptx::f2_add(acc0, ptx::f2_make(p0, p1));
                        pk[c] = ptx::pack_bf16(p0, p1);
                    }
                };
                auto publish = [&](int half) {
                    ptx::tmem_st_wait();
                    ptx::tc_fence_before();
                    ptx::mbar_arrive(&bar->p_full[t][half]);
                    if (row == 0) QVK_TRACE(512 + t * 256 + j * 8 + 2 + half);
                };
                // P half 0 (parts 0, 1) is published after part 2 has been computed, so the wait for its TMEM
                // stores overlaps 16 exponential pairs instead of stalling the warp.
                {
                    uint32_t pk[16];
                    part(0, pk);
                    QVK_TMEM_ST16(s_col + 0, pk);
                    part(1, pk);
                    QVK_TMEM_ST16(s_col + 16, pk);
                    part(2, pk);
                    publish(0);
                    QVK_TMEM_ST16(s_col + 32, pk);
                    part(3, pk);
                    QVK_TMEM_ST16(s_col + 48, pk);
                    publish(1);
                }
                float s0, s1, s2, s3;
                ptx::f2_split(acc0, s0, s1);
                ptx::f2_split(acc1, s2, s3);
                l += (s0 + s1) + (s2 + s3);
            }
            if (p.lse) {  // SnapKV's observation window = the group's last lse_window rows
                const int qpos = mt * kBM + row;
                const int r = qpos - (w.n - p.lse_window);
                if (qpos < w.n && r >= 0)
                    p.lse[(static_cast<int64_t>(w.g) * p.n_q + (t ? w.hq1 : w.hq0)) * p.lse_window + r] =
                        m_ref + __log2f(l);
            }
            if (units) ptx::mbar_wait(&bar->l_free[t], (units - 1) & 1);  // previous unit's sums consumed
            bar->row_sum[t][row] = l;
            ptx::mbar_arrive(&bar->l_full[t]);
            ++units;
            ++unit_iter;
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == kMmaWarp) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tmem);
    }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(tensor_map_encoder());
}

// (tokens, heads, 128) bf16 viewed as a 3-D tensor {d, heads, tokens}; box {64, 1, 128}, 128-byte swizzle.
bool make_map(CUtensorMap* m, const void* base, int heads, int64_t tokens, int kD) {
    auto enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(kD), static_cast<cuuint64_t>(heads),
                          static_cast<cuuint64_t>(tokens)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(kD) * 2, static_cast<cuuint64_t>(heads) * kD * 2};
    cuuint32_t box[3] = {64, 1, static_cast<cuuint32_t>(kBM)};
    cuuint32_t estr[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int D, int kPoly>
int launch_attention_d(cudaStream_t stream, const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
                       const CUtensorMap& mo, const AttnParams& prm, unsigned grid) {
    QVK_CUDA_CHECK(func_attr(reinterpret_cast<const void*>(attention_fwd_kernel<D, kPoly>),
                             cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_bytes<D>())));
    attention_fwd_kernel<D, kPoly><<<grid, kThreads, smem_bytes<D>(), stream>>>(mq, mk, mv, mo, prm);
    QVK_LAUNCH_CHECK();
    return QVK_OK;
}

}  // namespace

int launch_attention2(cudaStream_t, const qvk_groups*, const void*, const void*, const void*, int, int, float, void*);

// (defaults for the developer tools that include this file directly; capi.cu declares its own)
int launch_attention(cudaStream_t stream, const qvk_groups* g, const void* q, const void* k, const void* v, int n_q,
                     int n_kv, int d_h, float scale, void* o, float* lse = nullptr, int lse_window = 0) {
    if (d_h != 128 && d_h != 64) {
        set_error("attention: head_dim must be 64 or 128 (got " + std::to_string(d_h) + ")");
        return QVK_E_UNSUPPORTED;
    }
    if (n_q <= 0 || n_kv <= 0 || n_q % n_kv != 0) QVK_INVALID("attention: n_q must be a positive multiple of n_kv");
    if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v) |
         reinterpret_cast<uintptr_t>(o)) & 15)
        QVK_INVALID("attention: q/k/v/o must be 16-byte aligned");
    if (g->total_tokens == 0 || g->max_tokens == 0) return QVK_OK;
    if (g->total_tokens > 0x7fffffff) QVK_INVALID("attention: more than 2^31 token rows");
    if (lse && lse_window <= 0) QVK_INVALID("attention: window statistics need a window >= 1");
    if (d_h == 128 && !lse && env_knob("QVK_ATTN_2CTA", 0))  // CTA-pair variant (attention2.cu), opt-in while evaluated
        return launch_attention2(stream, g, q, k, v, n_q, n_kv, scale, o);
    CUtensorMap mq, mk, mv, mo;
    if (!make_map(&mq, q, n_q, g->total_tokens, d_h) || !make_map(&mk, k, n_kv, g->total_tokens, d_h) ||
        !make_map(&mv, v, n_kv, g->total_tokens, d_h) || !make_map(&mo, o, n_q, g->total_tokens, d_h)) {
        set_error("attention: cuTensorMapEncodeTiled failed");
        return QVK_E_CUDA;
    }
    AttnParams prm;
    prm.tok_off = g->tok_off_d;
    prm.n_groups = g->n_groups;
    prm.n_q = n_q;
    prm.n_kv = n_kv;
    const int64_t tiles = (g->max_tokens + kBM - 1) / kBM;
    if (tiles > 0x3fffffff) QVK_INVALID("attention: group too long");
    prm.tiles_max = static_cast<int>(tiles);
    prm.scale_log2 = scale * 1.4426950408889634f;
    prm.o = static_cast<__nv_bfloat16*>(o);
    static const int pre = env_knob("QVK_ATTN_PRE", 1) != 0;
    prm.pre_issue = pre;
    prm.lse = lse;
    prm.lse_window = lse_window;
    // Unit order: blocks of groups whose K/V (at the longest group) total ~32 MB, so a block's K/V stays L2-resident
    // while all its units run (C4: 4 groups of 8 MB; DRAM reads per C4 launch 27 -> ~10 GB, +2.5 % tokens/s under the
    // power cap, 1432 -> 1460 MHz).  QVK_ATTN_GBLOCK overrides (groups per block; 0 = automatic).
    static const int gblock_env = env_knob("QVK_ATTN_GBLOCK", 0);
    const int64_t kv_group = g->max_tokens * n_kv * d_h * 4;  // K + V bytes of the longest group
    const int64_t gb_auto = std::max<int64_t>(1, (int64_t{32} << 20) / std::max<int64_t>(kv_group, 1));
    prm.gblock = static_cast<int>(std::min<int64_t>(gblock_env > 0 ? gblock_env : gb_auto, g->n_groups));
    const int64_t units = static_cast<int64_t>((prm.tiles_max + 1) / 2) * g->n_groups * n_q;
    if (units > 0x7fffffff) QVK_INVALID("attention: too many work units");
    prm.total_units = static_cast<int>(units);
    const int sms = grid_sms();
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(units, sms));
    // Of every 16 exponential pairs, kPoly run on the FMA pipe (tuning knob QVK_ATTN_POLY = 0 | 1 | 2 | 3 | 4 | 6;
    // DESIGN.md §3.1): 2 and 4 are equal at boost clocks, 2 is ~0.5 % ahead inside the power-capped C4 step.
    static const int poly = [] {
        const int v = env_knob("QVK_ATTN_POLY", 2);
        return (v == 0 || v == 1 || v == 3 || v == 4 || v == 6) ? v : 2;
    }();
    if (d_h == 128) {
        switch (poly) {
            case 0: return launch_attention_d<128, 0>(stream, mq, mk, mv, mo, prm, grid);
            case 1: return launch_attention_d<128, 1>(stream, mq, mk, mv, mo, prm, grid);
            case 3: return launch_attention_d<128, 3>(stream, mq, mk, mv, mo, prm, grid);
            case 4: return launch_attention_d<128, 4>(stream, mq, mk, mv, mo, prm, grid);
            case 6: return launch_attention_d<128, 6>(stream, mq, mk, mv, mo, prm, grid);
            default: return launch_attention_d<128, 2>(stream, mq, mk, mv, mo, prm, grid);
        }
    }
    return poly ? launch_attention_d<64, 4>(stream, mq, mk, mv, mo, prm, grid)
                : launch_attention_d<64, 0>(stream, mq, mk, mv, mo, prm, grid);
}

}  // namespace qvk
