// Device/pinned memory helpers for the engine: chunked bump arenas (fronts are
// rebuilt wholesale every stage, so per-stage ping-pong arenas replace a
// general allocator) and a pinned staging area for descriptor uploads.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "spqr.h"

namespace spqr {

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) ::spqr::cuda_check((x), #x)

class DeviceArena {
public:
    explicit DeviceArena(size_t chunk = size_t(256) << 20) : chunk_(chunk) {}
    DeviceArena(const DeviceArena&) = delete;
    DeviceArena& operator=(const DeviceArena&) = delete;
    ~DeviceArena() {
        for (auto& c : chunks_) cudaFree(c.base);
    }
    void* alloc(size_t bytes) {
        bytes = (bytes + 255) & ~size_t(255);
        if (bytes == 0) bytes = 256;
        for (; cur_ < chunks_.size(); ++cur_) {
            Chunk& c = chunks_[cur_];
            if (c.used + bytes <= c.cap) {
                void* p = c.base + c.used;
                c.used += bytes;
                in_use_ += bytes;
                peak_ = std::max(peak_, in_use_);
                return p;
            }
        }
        Chunk c;
        c.cap = std::max(chunk_, bytes);
        CK(cudaMalloc(reinterpret_cast<void**>(&c.base), c.cap));
        c.used = bytes;
        chunks_.push_back(c);
        cur_ = chunks_.size() - 1;
        in_use_ += bytes;
        peak_ = std::max(peak_, in_use_);
        return c.base;
    }
    template <class T>
    T* alloc_n(size_t n) { return static_cast<T*>(alloc(sizeof(T) * n)); }
    void reset() {
        for (auto& c : chunks_) c.used = 0;
        cur_ = 0;
        in_use_ = 0;
    }
    size_t peak() const { return peak_; }
    // (base, used bytes) of every chunk, e.g. to mirror the arena on the host in a few copies
    template <class F>
    void for_each_chunk(F f) const {
        for (const auto& c : chunks_) f(c.base, c.used);
    }
    size_t reserved() const {
        size_t s = 0;
        for (auto& c : chunks_) s += c.cap;
        return s;
    }

private:
    struct Chunk { char* base = nullptr; size_t cap = 0, used = 0; };
    std::vector<Chunk> chunks_;
    size_t cur_ = 0, chunk_, in_use_ = 0, peak_ = 0;
};

// Pinned host staging; reset only after the stream has drained.
class PinnedArena {
public:
    explicit PinnedArena(size_t chunk = size_t(64) << 20) : chunk_(chunk) {}
    PinnedArena(const PinnedArena&) = delete;
    ~PinnedArena() {
        for (auto& c : chunks_) cudaFreeHost(c.base);
    }
    void* alloc(size_t bytes) {
        bytes = (bytes + 63) & ~size_t(63);
        if (bytes == 0) bytes = 64;
        for (; cur_ < chunks_.size(); ++cur_) {
            Chunk& c = chunks_[cur_];
            if (c.used + bytes <= c.cap) {
                void* p = c.base + c.used;
                c.used += bytes;
                return p;
            }
        }
        Chunk c;
        c.cap = std::max(chunk_, bytes);
        CK(cudaMallocHost(reinterpret_cast<void**>(&c.base), c.cap));
        c.used = bytes;
        chunks_.push_back(c);
        cur_ = chunks_.size() - 1;
        return c.base;
    }
    void reset() {
        for (auto& c : chunks_) c.used = 0;
        cur_ = 0;
    }

private:
    struct Chunk { char* base = nullptr; size_t cap = 0, used = 0; };
    std::vector<Chunk> chunks_;
    size_t cur_ = 0, chunk_;
};

// Large host copies (pinned staging <-> host vectors) split over the OpenMP
// threads: a single thread's memcpy is memory-latency bound far below DRAM speed.
inline void par_memcpy(void* dst, const void* src, size_t bytes) {
    constexpr size_t kChunk = size_t(64) << 10;
    if (bytes < 4 * kChunk) {
        std::memcpy(dst, src, bytes);
        return;
    }
    const long long n = static_cast<long long>((bytes + kChunk - 1) / kChunk);
#pragma omp parallel for schedule(static)
    for (long long c = 0; c < n; ++c) {
        const size_t off = static_cast<size_t>(c) * kChunk;
        std::memcpy(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off, std::min(kChunk, bytes - off));
    }
}

// Process-wide pinned staging for one-shot uploads (solve plans, matrices): pinning a fresh
// 64 MB buffer per call cost tens of ms.  Callers hold `mu` until their copies have completed;
// never destroyed (no CUDA calls during process teardown).
struct SharedPinned {
    std::mutex mu;
    PinnedArena arena;
    static SharedPinned& get() {
        static SharedPinned* s = new SharedPinned;
        return *s;
    }
};

// Uploads host vectors through pinned memory into a device arena.
struct Uploader {
    DeviceArena* dev;
    PinnedArena* pin;
    cudaStream_t st;
    size_t bytes_h2d = 0;
    template <class T>
    T* put(const T* h, size_t n) {
        if (n == 0) return nullptr;
        T* d = dev->alloc_n<T>(n);
        void* p = pin->alloc(sizeof(T) * n);
        par_memcpy(p, h, sizeof(T) * n);
        CK(cudaMemcpyAsync(d, p, sizeof(T) * n, cudaMemcpyHostToDevice, st));
        bytes_h2d += sizeof(T) * n;
        return d;
    }
    template <class T>
    T* put(const std::vector<T>& v) { return put(v.data(), v.size()); }
};

}  // namespace spqr
