// Shared host/device definitions for libpkgpu (B200, sm_100a).
#pragma once

#include <cstdint>
#include <cstdio>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include <cuda_runtime.h>

namespace pkgpu {

// Exception classes mirror the reference's (SURVEY.md §8b "Errors").
struct InvalidArgument : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct ConfigError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct RuntimeError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define PK_CUDA(x)                                                                                                  \
    do {                                                                                                            \
        cudaError_t e_ = (x);                                                                                       \
        if (e_ != cudaSuccess)                                                                                      \
            throw ::pkgpu::CudaError(std::string("CUDA error ") + cudaGetErrorString(e_) + " at " + __FILE__ + ":" + \
                                     std::to_string(__LINE__));                                                     \
    } while (0)

constexpr double kInner = 1.05; // include/pkifmm/geometry.hpp:17
constexpr double kOuter = 2.95; // include/pkifmm/geometry.hpp:18
constexpr int kMaxDepth = 12;   // src/fmm.cpp:301 default max_depth
constexpr int kNumM2L = 316;    // offsets 2 <= |d|_inf <= 3

inline int surface_point_count(int p) { return 6 * (p - 1) * (p - 1) + 2; }
inline int round_up(int x, int m) { return (x + m - 1) / m * m; }

// offset code of a cell offset d in [-3,3]^3 (src/fmm.cpp:51 uses the same packing)
__host__ __device__ inline int offset_code(int dx, int dy, int dz) { return (dx + 3) * 49 + (dy + 3) * 7 + (dz + 3); }
// image shift code of s in {-1,0,1}^3
__host__ __device__ inline int shift_code(int sx, int sy, int sz) { return (sx + 1) * 9 + (sy + 1) * 3 + (sz + 1); }
__host__ __device__ inline void shift_decode(int c, int &sx, int &sy, int &sz) {
    sx = c / 9 - 1;
    sy = (c / 3) % 3 - 1;
    sz = c % 3 - 1;
}

// Grow-only device buffer (workspace reuse across evaluate calls).
struct DevBuf {
    void *ptr = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    ~DevBuf() {
        if (ptr) cudaFree(ptr);
    }
    void *reserve(size_t b) {
        if (b > bytes) {
            if (ptr) PK_CUDA(cudaFree(ptr));
            ptr = nullptr;
            const size_t nb = std::max(b, bytes + bytes / 4);
            PK_CUDA(cudaMalloc(&ptr, nb));
            bytes = nb;
        }
        return ptr;
    }
    template <class T> T *as(size_t n) { return static_cast<T *>(reserve(sizeof(T) * std::max<size_t>(n, 1))); }
};

// Named workspace pool owned by a context.
struct Workspace {
    std::unordered_map<std::string, std::unique_ptr<DevBuf>> bufs;
    template <class T> T *get(const std::string &name, size_t n) {
        auto &b = bufs[name];
        if (!b) b = std::make_unique<DevBuf>();
        return b->as<T>(n);
    }
};

inline unsigned blocks_for(size_t n, unsigned threads) { return static_cast<unsigned>((n + threads - 1) / threads); }

} // namespace pkgpu
