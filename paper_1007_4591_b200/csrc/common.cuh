// common.cuh -- shared internals of libfmmbem (CUDA path only; never the oracle).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/fmmbem.h"

namespace fmm {

// Error carried from deep inside the library to the ABI boundary.
struct Error : std::runtime_error {
  fmmbem_status code;
  Error(fmmbem_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define FMM_CUDA(call)                                                                                    \
  do {                                                                                                    \
    cudaError_t e_ = (call);                                                                              \
    if (e_ != cudaSuccess)                                                                                \
      throw ::fmm::Error(e_ == cudaErrorMemoryAllocation ? FMMBEM_E_NOMEM : FMMBEM_E_CUDA,                \
                         std::string(#call) + ": " + cudaGetErrorString(e_) + " (" + __FILE__ + ":" +     \
                             std::to_string(__LINE__) + ")");                                             \
  } while (0)

#define FMM_CHECK_LAUNCH() FMM_CUDA(cudaGetLastError())

// Owned device buffer.
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) {
    o.p = nullptr;
    o.n = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      n = o.n;
      o.p = nullptr;
      o.n = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    if (count == n && p) return;
    release();
    if (count) FMM_CUDA(cudaMalloc(&p, count * sizeof(T)));
    n = count;
  }
  void zero(cudaStream_t s) {
    if (n) FMM_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
  T* get() const { return p; }
  size_t bytes() const { return n * sizeof(T); }
};

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

constexpr int MAX_LEVEL = 21;  // 3 x 21 bits in a 64-bit Morton key
constexpr int MAX_TERMS = 16;

// Morton helpers: x least significant within each triple.
__host__ __device__ inline uint64_t spread3(uint32_t v) {
  uint64_t x = v & 0x1fffff;
  x = (x | x << 32) & 0x1f00000000ffffULL;
  x = (x | x << 16) & 0x1f0000ff0000ffULL;
  x = (x | x << 8) & 0x100f00f00f00f00fULL;
  x = (x | x << 4) & 0x10c30c30c30c30c3ULL;
  x = (x | x << 2) & 0x1249249249249249ULL;
  return x;
}
__host__ __device__ inline uint32_t compact3(uint64_t x) {
  x &= 0x1249249249249249ULL;
  x = (x ^ (x >> 2)) & 0x10c30c30c30c30c3ULL;
  x = (x ^ (x >> 4)) & 0x100f00f00f00f00fULL;
  x = (x ^ (x >> 8)) & 0x1f0000ff0000ffULL;
  x = (x ^ (x >> 16)) & 0x1f00000000ffffULL;
  x = (x ^ (x >> 32)) & 0x1fffffULL;
  return (uint32_t)x;
}
__host__ __device__ inline uint64_t morton(uint32_t ix, uint32_t iy, uint32_t iz) {
  return spread3(ix) | (spread3(iy) << 1) | (spread3(iz) << 2);
}
__host__ __device__ inline void demorton(uint64_t k, int& ix, int& iy, int& iz) {
  ix = (int)compact3(k);
  iy = (int)compact3(k >> 1);
  iz = (int)compact3(k >> 2);
}

}  // namespace fmm
