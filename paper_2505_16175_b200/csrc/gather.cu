// (a10)/(a11) KV compaction: copy the retained (token, head) rows of K and V into the persistent cache at their
// static offsets, and write the global token ids (prefill.cpp:277-280 gather, :304-308 cache append).
//
// The grid walks the DESTINATION (cache) linearly in 16-byte vectors, so stores are perfectly coalesced and every
// source row (width * elem bytes, 256 B for bf16 d_h = 128) is read as whole contiguous 32-byte sectors.
// Algorithmic bytes per retained (row, head): 2 * width * elem (read K, V) + 2 * width * elem (write) + 8 (origin).
#include "common.cuh"

namespace qvk {
namespace {

template <typename V>
__global__ void __launch_bounds__(256) gather_kernel(const uint8_t* __restrict__ k, const uint8_t* __restrict__ v,
                                                     int row_bytes, int heads, int n_groups,
                                                     const int64_t* __restrict__ tok_off,
                                                     const int64_t* __restrict__ row_off,
                                                     const uint64_t* __restrict__ first_token,
                                                     const uint32_t* __restrict__ idx, int64_t total_units,
                                                     int64_t keep_stride,
                                                     uint8_t* __restrict__ kc, uint8_t* __restrict__ vc,
                                                     uint64_t* __restrict__ origin, uint32_t* __restrict__ idx_out) {
    const int vec_per_unit = row_bytes / static_cast<int>(sizeof(V));
    const int64_t total = total_units * vec_per_unit;
    for (int64_t w = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; w < total;
         w += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t cu = w / vec_per_unit;        // cache unit = cache_row * heads + head
        const int part = static_cast<int>(w - cu * vec_per_unit);
        const int64_t row = cu / heads;
        const int h = static_cast<int>(cu - row * heads);
        const int g = find_group_fast(row_off, n_groups, row, keep_stride);
        const int64_t r = row - __ldg(row_off + g);
        const int64_t src_tok = idx ? static_cast<int64_t>(__ldg(idx + cu)) : r;
        const int64_t src_unit = (__ldg(tok_off + g) + src_tok) * heads + h;
        const int64_t so = src_unit * row_bytes + static_cast<int64_t>(part) * sizeof(V);
        const int64_t dof = cu * row_bytes + static_cast<int64_t>(part) * sizeof(V);
        const V a = __ldg(reinterpret_cast<const V*>(k + so));
        const V b = __ldg(reinterpret_cast<const V*>(v + so));
        *reinterpret_cast<V*>(kc + dof) = a;
        *reinterpret_cast<V*>(vc + dof) = b;
        if (origin && part == 0) origin[cu] = __ldg(first_token + g) + static_cast<uint64_t>(src_tok);
        if (idx_out && part == 0) idx_out[cu] = static_cast<uint32_t>(src_tok);  // identity path: r = 0..keep-1
    }
}

}  // namespace

// keep_stride: cache rows of a full-size group when known (rho given), else 0 = derive / binary search.
// idx_out (identity path only, idx == NULL): receives the retained local indices 0..keep-1 like every scored path.
int launch_gather(cudaStream_t stream, const qvk_groups* g, const void* k, const void* v, int dtype, int heads,
                  int width, const uint32_t* idx, void* kc, void* vc, uint64_t* origin, int64_t keep_stride,
                  uint32_t* idx_out) {
    if (origin && !g->first_token_d) QVK_INVALID("gather: origin requested without first_token");
    if (keep_stride <= 0 && g->n_groups > 0 && g->total_rows % g->n_groups == 0)
        keep_stride = g->total_rows / g->n_groups;  // equal groups
    const int elem = dtype == QVK_F32 ? 4 : 2;
    const int row_bytes = width * elem;
    const int64_t units = g->total_rows * heads;
    if (units == 0) return QVK_OK;
    const uintptr_t align = reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v) |
                            reinterpret_cast<uintptr_t>(kc) | reinterpret_cast<uintptr_t>(vc);
    int vec = 2;
    if (row_bytes % 16 == 0 && (align & 15) == 0) vec = 16;
    else if (row_bytes % 4 == 0 && (align & 3) == 0) vec = 4;
    const int64_t total = units * (row_bytes / vec);
    const int64_t want = (total + 255) / 256;
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>(want, static_cast<int64_t>(kNumSms) * 16));
    auto args = [&](auto* kern) {
        kern<<<blocks, 256, 0, stream>>>(static_cast<const uint8_t*>(k), static_cast<const uint8_t*>(v), row_bytes,
                                         heads, g->n_groups, g->tok_off_d, g->row_off_d, g->first_token_d, idx,
                                         units, keep_stride, static_cast<uint8_t*>(kc), static_cast<uint8_t*>(vc),
                                         origin, idx ? nullptr : idx_out);
    };
    if (vec == 16) args(gather_kernel<uint4>);
    else if (vec == 4) args(gather_kernel<uint32_t>);
    else args(gather_kernel<uint16_t>);
    QVK_LAUNCH_CHECK();
    return QVK_OK;
}

}  // namespace qvk
