// Shared device/host helpers for the qvk library (sm_100a only).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>

#include "qvk.h"

namespace qvk {

// Thread-local error text returned by qvk_last_error() (capi.cu).
void set_error(const std::string& msg);

// Stream-ordered scratch allocation (cudaMallocAsync) from the device's default memory pool, whose release threshold
// is raised once per device so freed scratch stays pooled across stream synchronisations (with the default
// threshold of 0 every synchronise returns it to the driver and the next call pays a real allocation, ~0.4 ms).
cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t stream);

// cudaFuncSetAttribute(func, attr, value) once per (function, device, attribute) — raised when a larger value is
// asked for; attributes are per device, and one process may drive several GPUs.
cudaError_t func_attr(const void* func, cudaFuncAttribute attr, int value);

// Process-wide lookups, initialised once in a thread-safe way (capi.cu): the SM count of the current device at first
// use, an integer tuning knob from the environment (default when unset), and the driver's cuTensorMapEncodeTiled.
int sm_count();
int grid_sms();  // sm_count() minus the SMs reserved for concurrent work (qvk_reserve_sms)
int env_knob(const char* name, int def);
void* tensor_map_encoder();  // PFN_cuTensorMapEncodeTiled_v12000, or nullptr

constexpr int kNumSms = 148;

// Order-preserving map of a double score onto uint64: larger score <=> larger key.  -0.0 is canonicalised to +0.0
// first because the reference compares scores with `!=` (prefill.cpp:245), under which the two zeros tie.
__device__ __forceinline__ uint64_t score_key(double s) {
    if (s == 0.0) s = 0.0;
    const uint64_t u = static_cast<uint64_t>(__double_as_longlong(s));
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

// Group containing token row t: largest g with off[g] <= t (off has G+1 ascending entries).
__device__ __forceinline__ int find_group(const int64_t* __restrict__ off, int n_groups, int64_t t) {
    int lo = 0, hi = n_groups - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (__ldg(off + mid) <= t) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// Same, for the usual case of equal group sizes: guess g = t / stride (stride = the largest group's size) and verify
// with two independent loads; fall back to the search for ragged plans.  32-bit division when t, stride fit.
__device__ __forceinline__ int find_group_fast(const int64_t* __restrict__ off, int n_groups, int64_t t,
                                               int64_t stride) {
    if (stride > 0 && t < 0x7fffffff && stride < 0x7fffffff) {
        uint32_t g = static_cast<uint32_t>(t) / static_cast<uint32_t>(stride);
        if (g > static_cast<uint32_t>(n_groups - 1)) g = n_groups - 1;
        if (__ldg(off + g) <= t && t < __ldg(off + g + 1)) return static_cast<int>(g);
    }
    return find_group(off, n_groups, t);
}

__device__ __forceinline__ uint64_t splitmix64_at(uint64_t state0, uint64_t i) {
    // Draw i (0-based) of splitmix64 seeded with state0 (synthetic.cpp:5-10): state advances by gamma per draw.
    uint64_t z = state0 + (i + 1) * 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t stream_seed(uint64_t seed, uint32_t tag, uint32_t layer) {
    // prefill.cpp:13-18
    uint64_t s = seed;
    s = s * 0x100000001b3ull + tag + 1;
    s = s * 0x100000001b3ull + layer + 1;
    return s;
}

}  // namespace qvk

#define QVK_CUDA_CHECK(expr)                                                                    \
    do {                                                                                        \
        cudaError_t _e = (expr);                                                                \
        if (_e != cudaSuccess) {                                                                \
            ::qvk::set_error(std::string("CUDA error: ") + cudaGetErrorString(_e) + " at " +    \
                             __FILE__ + ":" + std::to_string(__LINE__));                        \
            return QVK_E_CUDA;                                                                  \
        }                                                                                       \
    } while (0)

#define QVK_LAUNCH_CHECK() QVK_CUDA_CHECK(cudaGetLastError())

#define QVK_INVALID(msg)              \
    do {                              \
        ::qvk::set_error(msg);        \
        return QVK_E_INVALID;         \
    } while (0)
