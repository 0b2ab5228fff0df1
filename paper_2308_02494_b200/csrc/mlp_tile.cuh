// SIMT building blocks for the 64-point tile MLP (decoder of model.py:152-162
// and its backward, optim.py:116-127).  A CTA of 256 threads (8 warps) owns a
// tile of P = 64 points whose activations live in shared memory.  Thread
// mapping for the 64-wide layers: lane -> points {lane, lane+32}, warp w ->
// hidden units [8w, 8w+8): weight loads are warp-uniform (one broadcast per
// warp) and activation loads are conflict-free (odd row strides).
#pragma once

#include "common.cuh"

namespace apmg {

constexpr int kTileP = 64;
constexpr int kTileThreads = 256;
constexpr int kHidden = 64;
constexpr int kHS = kHidden + 1;  // smem row stride of hidden activations

__host__ __device__ inline int feat_stride(int F) { return (F % 2 == 0) ? F + 1 : F; }

// sO[p][j] = act(sum_k sA[p][k] * W[j*K + k]) for p < 64, j < 64.
template <typename T>
__device__ __forceinline__ void tile_dense(const T* sA, int as, int K, const T* __restrict__ W, T* sO, int os,
                                           bool relu) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T acc0[8], acc1[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc0[j] = acc1[j] = T(0);
  const T* a0 = sA + lane * as;
  const T* a1 = sA + (lane + 32) * as;
  const T* wr = W + int64_t(8 * w) * K;
#pragma unroll 4
  for (int k = 0; k < K; ++k) {
    const T f0 = a0[k], f1 = a1[k];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const T wv = ldg(wr + j * K + k);
      acc0[j] = fma(f0, wv, acc0[j]);
      acc1[j] = fma(f1, wv, acc1[j]);
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    T v0 = acc0[j], v1 = acc1[j];
    if (relu) {
      v0 = v0 > T(0) ? v0 : T(0);
      v1 = v1 > T(0) ? v1 : T(0);
    }
    sO[lane * os + 8 * w + j] = v0;
    sO[(lane + 32) * os + 8 * w + j] = v1;
  }
}

// raw[p] = sum_j sH2[p][j] * w3[j]; out = raw * span + vmin (threads 0..63).
template <typename T>
__device__ __forceinline__ T tile_head(const T* sH2, const T* __restrict__ w3, int p, T span, T vmin) {
  T acc = T(0);
#pragma unroll 8
  for (int j = 0; j < kHidden; ++j) acc = fma(sH2[p * kHS + j], ldg(w3 + j), acc);
  return add_rn(mul_rn(acc, span), vmin);
}

}  // namespace apmg
