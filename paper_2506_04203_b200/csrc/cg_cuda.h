// CUDA error plumbing and small device-buffer helpers (host side).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <stdexcept>
#include <string>

namespace cg {

// Engine error carrying a cg_status code (CG_ERR_* / cascade::Errc value).
struct EngineError : std::runtime_error {
    int code;
    EngineError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess)
        throw EngineError(100, std::string("CUDA error: ") + cudaGetErrorString(e) + " at " +
                                   what + " (" + file + ":" + std::to_string(line) + ")");
}

#define CG_CUDA(x) ::cg::cuda_check((x), #x, __FILE__, __LINE__)
#define CG_LAUNCH_CHECK() ::cg::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

// Grow-only device scratch buffer.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    void* reserve(size_t b) {
        if (b > bytes) {
            if (p) CG_CUDA(cudaFree(p));
            p = nullptr;
            size_t nb = b + b / 4 + 256;
            CG_CUDA(cudaMalloc(&p, nb));
            bytes = nb;
        }
        return p;
    }
    template <class T>
    T* as(size_t count) {
        return static_cast<T*>(reserve(count * sizeof(T) + 16));
    }
};

// Grow-only pinned host buffer.
struct HostBuf {
    void* p = nullptr;
    size_t bytes = 0;
    HostBuf() = default;
    HostBuf(const HostBuf&) = delete;
    HostBuf& operator=(const HostBuf&) = delete;
    ~HostBuf() {
        if (p) cudaFreeHost(p);
    }
    void* reserve(size_t b) {
        if (b > bytes) {
            if (p) CG_CUDA(cudaFreeHost(p));
            p = nullptr;
            size_t nb = b + b / 4 + 256;
            CG_CUDA(cudaMallocHost(&p, nb));
            bytes = nb;
        }
        return p;
    }
    template <class T>
    T* as(size_t count) {
        return static_cast<T*>(reserve(count * sizeof(T) + 16));
    }
};

}  // namespace cg
