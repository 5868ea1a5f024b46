// Shared host/device plumbing for libdouble_b200: status/exception mapping, CUDA checks, small
// device helpers.  Host code throws dbl::Error (carrying a dbl_status); the C-ABI boundary in
// capi.cu converts it to a status + thread-local message.
#pragma once
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only; the ranges cost nothing unless a profiler is attached

#include <cstdint>
#include <stdexcept>
#include <string>

#include "double_b200.h"

namespace dbl {

struct Error : std::runtime_error {
    dbl_status status;
    Error(dbl_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] inline void throw_invalid(const std::string& m) { throw Error(DBL_INVALID_ARGUMENT, m); }
[[noreturn]] inline void throw_runtime(const std::string& m) { throw Error(DBL_RUNTIME_ERROR, m); }
[[noreturn]] inline void throw_logic(const std::string& m) { throw Error(DBL_LOGIC_ERROR, m); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess) {
        throw Error(DBL_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e) + " (" + file +
                                        ":" + std::to_string(line) + ")");
    }
}
#define CUDA_CHECK(x) ::dbl::cuda_check((x), #x, __FILE__, __LINE__)
// every kernel launch in the library is followed by CUDA_LAUNCH_CHECK(), which also counts it
// (dbl_run_metrics::kernel_launches, bench.py's gpu_launches)
long long& launch_counter();
#define CUDA_LAUNCH_CHECK()                                                                  \
    do {                                                                                     \
        ::dbl::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__);          \
        ++::dbl::launch_counter();                                                           \
    } while (0)

// RAII device buffer
template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    explicit DevBuf(size_t count) { alloc(count); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(size_t count) {
        release();
        if (count) CUDA_CHECK(cudaMalloc(&p, count * sizeof(T)));
        n = count;
    }
    // s == 0: completes before returning — the decode loop's streams are non-blocking, so an
    // asynchronous legacy-stream memset could land after their first writes to this buffer
    void zero(cudaStream_t s = 0) {
        if (!n) return;
        CUDA_CHECK(cudaMemsetAsync(p, 0, n * sizeof(T), s));
        if (s == 0) CUDA_CHECK(cudaStreamSynchronize(0));
    }
    void release() { if (p) cudaFree(p); p = nullptr; n = 0; }
    size_t bytes() const { return n * sizeof(T); }
};

// Process-wide cache of mapped pinned host blocks (power-of-two size classes).  Pinning pages costs
// milliseconds per MiB; every run()/store call needs a few such buffers, so freed blocks are kept
// for reuse (callers only release a block after the device is done with it).
void* pinned_get(size_t bytes, size_t* got);
void pinned_put(void* p, size_t bytes);

// RAII pinned host buffer (mapped: dev() aliases it on the device)
template <class T>
struct PinBuf {
    T* p = nullptr;
    size_t n = 0;
    size_t cap_bytes = 0;
    PinBuf() = default;
    explicit PinBuf(size_t count) { alloc(count); }
    PinBuf(const PinBuf&) = delete;
    PinBuf& operator=(const PinBuf&) = delete;
    ~PinBuf() { release(); }
    void release() {
        if (p) pinned_put(p, cap_bytes);
        p = nullptr;
        n = 0;
        cap_bytes = 0;
    }
    void alloc(size_t count) {
        release();
        if (count) p = static_cast<T*>(pinned_get(count * sizeof(T), &cap_bytes));
        n = count;
    }
    T* dev() const {  // device alias of the mapped pinned allocation
        void* d = nullptr;
        CUDA_CHECK(cudaHostGetDevicePointer(&d, p, 0));
        return static_cast<T*>(d);
    }
};

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        CUDA_CHECK(cudaGetDevice(&prev));
        if (prev != dev) CUDA_CHECK(cudaSetDevice(dev));
    }
    ~DeviceGuard() { if (prev >= 0) cudaSetDevice(prev); }
};

// NVTX range over a host scope (nsys / ncu --nvtx show the decode loop's stages: "dbl.round",
// "dbl.draft", "dbl.target", "dbl.wait", "dbl.finish_round", "dbl.ar_block", ...)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

void require_device(int device);  // throws DBL_CUDA_ERROR unless an sm_100 device is usable

constexpr int kMaxOrder = 8;      // datastore n-gram order bound (reference default N = 3)

}  // namespace dbl
