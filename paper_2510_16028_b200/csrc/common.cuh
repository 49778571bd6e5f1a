// Shared helpers for the NAO B200 kernels (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>

#include "../../include/nao_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "paper_2510_16028_b200 kernels are written for sm_100a only"
#endif

namespace nao {

constexpr int kNumSMs = 148;

// Per-thread last-error text (nao_last_error).
void set_error(const char* fmt, ...);

#define NAO_CHECK_CUDA(expr)                                                    \
    do {                                                                        \
        cudaError_t _e = (expr);                                                \
        if (_e != cudaSuccess) {                                                \
            ::nao::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,          \
                             cudaGetErrorString(_e));                           \
            return NAO_ECUDA;                                                   \
        }                                                                       \
    } while (0)

#define NAO_CHECK_LAUNCH()                                                      \
    do {                                                                        \
        cudaError_t _e = cudaGetLastError();                                    \
        if (_e != cudaSuccess) {                                                \
            ::nao::set_error("%s:%d launch: %s", __FILE__, __LINE__,            \
                             cudaGetErrorString(_e));                           \
            return NAO_ECUDA;                                                   \
        }                                                                       \
    } while (0)

#define NAO_REQUIRE(cond, ...)                                                  \
    do {                                                                        \
        if (!(cond)) {                                                          \
            ::nao::set_error(__VA_ARGS__);                                      \
            return NAO_EINVAL;                                                  \
        }                                                                       \
    } while (0)

// Simple bump allocator over the caller-provided workspace.
struct Workspace {
    uint8_t* base;
    size_t size;
    size_t used = 0;
    __host__ Workspace(void* b, size_t s) : base(static_cast<uint8_t*>(b)), size(s) {}
    template <typename T>
    __host__ T* take(size_t count, size_t align = 256) {
        size_t off = (used + align - 1) / align * align;
        size_t bytes = count * sizeof(T);
        if (base == nullptr || off + bytes > size) return nullptr;
        used = off + bytes;
        return reinterpret_cast<T*>(base + off);
    }
};

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

// Non-negative doubles order like their bit patterns.
__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
    atomicMax(reinterpret_cast<unsigned long long*>(addr),
              static_cast<unsigned long long>(__double_as_longlong(v)));
}
__device__ __forceinline__ void atomic_min_nonneg(double* addr, double v) {
    atomicMin(reinterpret_cast<unsigned long long*>(addr),
              static_cast<unsigned long long>(__double_as_longlong(v)));
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

}  // namespace nao
