// Staged copies between pageable host memory and the device (include/qvk.h qvk_memcpy_{d2h,h2d}_pageable).
//
// The reference's API hands the path std::vectors (pageable memory).  A plain cudaMemcpy from / to pageable memory
// goes through the driver's own small bounce buffer one piece at a time (measured 2.1 GB/s D2H, 11 GB/s H2D on the
// B200 box, tools/exact_bench.py).  Here the copy is split into 32 MB chunks through two pinned staging buffers:
// the DMA of chunk i+1 (55 GB/s) runs while kHostThreads threads copy chunk i between the staging buffer and the
// caller's memory, so the copy runs at the host's memcpy bandwidth.  One staging pair per process (mutex).
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"

namespace qvk {
namespace {

constexpr size_t kChunk = size_t(32) << 20;
constexpr size_t kDirect = size_t(4) << 20;  // below this a plain copy is as fast
constexpr int kHostThreads = 8;

struct Staging {
    std::mutex mu;
    void* buf[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    int dev = -1;
};

Staging& staging() {
    static auto* s = new Staging();  // leaked: pinned memory must not be freed from a static destructor
    return *s;
}

cudaError_t ensure(Staging& st) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (st.buf[0] && st.dev == dev) return cudaSuccess;
    for (int i = 0; i < 2; ++i) {
        if (!st.buf[i] && (e = cudaHostAlloc(&st.buf[i], kChunk, cudaHostAllocPortable)) != cudaSuccess) return e;
        if (st.ev[i]) cudaEventDestroy(st.ev[i]);
        if ((e = cudaEventCreateWithFlags(&st.ev[i], cudaEventDisableTiming)) != cudaSuccess) return e;
    }
    st.dev = dev;
    return cudaSuccess;
}

void par_memcpy(void* dst, const void* src, size_t n) {
    if (n < (size_t(2) << 20)) {
        std::memcpy(dst, src, n);
        return;
    }
    std::thread th[kHostThreads];
    const size_t per = (n + kHostThreads - 1) / kHostThreads;
    for (int t = 0; t < kHostThreads; ++t) {
        const size_t a = std::min(n, t * per), b = std::min(n, a + per);
        th[t] = std::thread([=] { std::memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a); });
    }
    for (auto& t : th) t.join();
}

}  // namespace
}  // namespace qvk

using namespace qvk;

extern "C" {

int qvk_memcpy_d2h_pageable(void* dst, const void* src, size_t bytes, qvk_stream_t s) {
    if (!bytes) return QVK_OK;
    if (bytes <= kDirect) {
        QVK_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
        QVK_CUDA_CHECK(cudaStreamSynchronize(s));
        return QVK_OK;
    }
    Staging& st = staging();
    std::lock_guard<std::mutex> lk(st.mu);
    QVK_CUDA_CHECK(ensure(st));
    const size_t chunks = (bytes + kChunk - 1) / kChunk;
    auto issue = [&](size_t i) -> cudaError_t {
        const size_t off = i * kChunk, n = std::min(kChunk, bytes - off);
        cudaError_t e = cudaMemcpyAsync(st.buf[i & 1], static_cast<const char*>(src) + off, n,
                                        cudaMemcpyDeviceToHost, s);
        return e == cudaSuccess ? cudaEventRecord(st.ev[i & 1], s) : e;
    };
    QVK_CUDA_CHECK(issue(0));
    if (chunks > 1) QVK_CUDA_CHECK(issue(1));
    for (size_t i = 0; i < chunks; ++i) {
        QVK_CUDA_CHECK(cudaEventSynchronize(st.ev[i & 1]));
        const size_t off = i * kChunk, n = std::min(kChunk, bytes - off);
        par_memcpy(static_cast<char*>(dst) + off, st.buf[i & 1], n);
        if (i + 2 < chunks) QVK_CUDA_CHECK(issue(i + 2));
    }
    return QVK_OK;
}

int qvk_memcpy_h2d_pageable(void* dst, const void* src, size_t bytes, qvk_stream_t s) {
    if (!bytes) return QVK_OK;
    if (bytes <= kDirect) {
        QVK_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
        QVK_CUDA_CHECK(cudaStreamSynchronize(s));
        return QVK_OK;
    }
    Staging& st = staging();
    std::lock_guard<std::mutex> lk(st.mu);
    QVK_CUDA_CHECK(ensure(st));
    const size_t chunks = (bytes + kChunk - 1) / kChunk;
    for (size_t i = 0; i < chunks; ++i) {
        const size_t off = i * kChunk, n = std::min(kChunk, bytes - off);
        if (i >= 2) QVK_CUDA_CHECK(cudaEventSynchronize(st.ev[i & 1]));  // the DMA out of this buffer is done
        par_memcpy(st.buf[i & 1], static_cast<const char*>(src) + off, n);
        QVK_CUDA_CHECK(cudaMemcpyAsync(static_cast<char*>(dst) + off, st.buf[i & 1], n, cudaMemcpyHostToDevice, s));
        QVK_CUDA_CHECK(cudaEventRecord(st.ev[i & 1], s));
    }
    QVK_CUDA_CHECK(cudaStreamSynchronize(s));
    return QVK_OK;
}

}  // extern "C"
