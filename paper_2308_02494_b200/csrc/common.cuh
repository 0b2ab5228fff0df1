// Shared helpers for libapmg_cuda: error reporting, launch accounting,
// per-kernel CUDA-event timing and round-to-nearest arithmetic wrappers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <atomic>
#include <string>

#include "../../include/apmg_cuda.h"

namespace apmg {

void set_error(const char* fmt, ...);
std::atomic<uint64_t>& launch_counter();
bool kernel_timing_on();  // per-launch CUDA events active (apmg_kernel_timing_enable)

// Records a CUDA event pair around a launch when timing is enabled.
struct LaunchScope {
  const char* name;
  cudaStream_t stream;
  void* start = nullptr;
  LaunchScope(const char* n, cudaStream_t s);
  ~LaunchScope();
};

int num_sms();
// large-buffer cache (runtime.cu): blocks keep their allocation size for pool_free
void* pool_alloc(size_t bytes);
void pool_free(void* p, size_t bytes);
void release_pool();
size_t pool_cached_bytes();  // bytes held by the cache (free for reuse)
// stream-ordered scratch (runtime.cu)
void* stream_alloc(size_t bytes, cudaStream_t st);
void stream_free(void* p, cudaStream_t st);
// owns one stream-ordered scratch block: freed on every exit path of the launcher
struct StreamScratch {
  void* p = nullptr;
  cudaStream_t st = nullptr;
  StreamScratch() = default;
  StreamScratch(size_t bytes, cudaStream_t s) : p(stream_alloc(bytes, s)), st(s) {}
  StreamScratch(const StreamScratch&) = delete;
  StreamScratch& operator=(const StreamScratch&) = delete;
  StreamScratch& operator=(StreamScratch&& o) noexcept {
    if (this != &o) {
      stream_free(p, st);
      p = o.p;
      st = o.st;
      o.p = nullptr;
    }
    return *this;
  }
  ~StreamScratch() { stream_free(p, st); }
  template <typename U>
  U* as() const {
    return static_cast<U*>(p);
  }
};

#define APMG_CUDA_TRY(expr)                                                                  \
  do {                                                                                       \
    cudaError_t _e = (expr);                                                                 \
    if (_e != cudaSuccess) {                                                                 \
      ::apmg::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
      return APMG_E_CUDA;                                                                    \
    }                                                                                        \
  } while (0)

#define APMG_ARG_CHECK(cond, ...)      \
  do {                                 \
    if (!(cond)) {                     \
      ::apmg::set_error(__VA_ARGS__);  \
      return APMG_E_ARG;               \
    }                                  \
  } while (0)

// Launch a kernel with accounting; returns APMG_E_CUDA from the enclosing function on error.
#define APMG_LAUNCH(name, kernel, grid, block, smem, stream, ...)                            \
  do {                                                                                       \
    {                                                                                        \
      ::apmg::LaunchScope _ls(name, stream);                                                 \
      kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);                            \
    }                                                                                        \
    ::apmg::launch_counter().fetch_add(1, std::memory_order_relaxed);                        \
    cudaError_t _e = cudaGetLastError();                                                     \
    if (_e != cudaSuccess) {                                                                 \
      ::apmg::set_error("launch %s: %s", name, cudaGetErrorString(_e));                      \
      return APMG_E_CUDA;                                                                    \
    }                                                                                        \
  } while (0)

// ---- explicit round-to-nearest arithmetic (no FMA contraction) so the
// elementwise numpy expressions of the reference are reproduced bit for bit.
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float sqrt_rn(float a) { return __fsqrt_rn(a); }
__device__ __forceinline__ double sqrt_rn(double a) { return __dsqrt_rn(a); }

template <typename T>
__device__ __forceinline__ T ldg(const T* p) {
  return __ldg(p);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide f64 sum; every thread gets the result. `scratch` >= 32 doubles.
__device__ __forceinline__ double block_sum(double v, double* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  double t = (threadIdx.x < nw) ? scratch[threadIdx.x] : 0.0;
  if (warp == 0) t = warp_sum(t);
  if (threadIdx.x == 0) scratch[0] = t;
  __syncthreads();
  double r = scratch[0];
  __syncthreads();
  return r;
}

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Bump allocator over a caller-provided device workspace.
struct Carver {
  char* base;
  size_t cap, used = 0;
  Carver(void* b, size_t c) : base(static_cast<char*>(b)), cap(c) {}
  template <typename T>
  T* take(size_t count) {
    used = align_up(used, 256);
    T* p = reinterpret_cast<T*>(base ? base + used : nullptr);
    used += count * sizeof(T);
    return p;
  }
  bool ok() const { return used <= cap; }
};

}  // namespace apmg
