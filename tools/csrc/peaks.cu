// Peak probes for the per-kernel rooflines SURVEY 8(d) asks for (L2 gather, L2 RED, FP32,
// FP64, tcgen05 kind::tf32).  Each probe is one launch over the whole GPU; the host times
// it with CUDA events (tools/peaks.py) and divides the work returned in *work.
//   kind 0  L2 gather: random float2 loads from a `table_bytes` table (L2-resident when
//           <= ~100 MiB), the encoder's access unit; work = bytes loaded
//   kind 1  L2 RED: random float2 red.global.add into the table, the scatter's unit;
//           work = float2 REDs issued
//   kind 2  FP32 FFMA; work = FLOP
//   kind 3  FP64 DFMA; work = FLOP
//   kind 4  tcgen05.mma kind::tf32, M=128 N=256 K=8, back to back from one thread per CTA
//           (operands in smem, contents irrelevant); work = FLOP
//   kind 5  warp shuffles (__shfl_sync, 32-bit); work = shuffle instructions (per warp)
//   kind 7  L2 gather of random float4 (16-byte) elements; work = bytes loaded
//   kind 9  tcgen05.mma kind::f16 (bf16), K=16, M = 128 (64 if table_bytes >= 1000), N =
//           table_bytes % 1000, back to back into one accumulator, or M=128 N=64 alternating
//           over 4 accumulators (table_bytes = 1):
//           the per-instruction cost of the small products the MLP kernels issue; work = FLOP
//   kind 8  L2 RED of random float4 (red.global.add.v4.f32); work = float4 REDs issued
//   kind 10 L2 gather of random 32-byte elements (ld.global.nc.v8.f32, LDG.E.ENL2.256); work = bytes
//   kind 6  shared-memory float atomic adds (red.shared.add.f32), 32 distinct banks per
//           instruction; work = atomic instructions (per warp)
#include "common.cuh"
#include "umma.cuh"

namespace apmg {

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

__global__ void __launch_bounds__(256) k_peak_gather(const float2* __restrict__ t, uint32_t mask, int iters,
                                                     float* __restrict__ sink) {
  uint32_t s = mix32(blockIdx.x * blockDim.x + threadIdx.x);
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    float2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      s = s * 1664525u + 1013904223u;
      v[u] = __ldg(t + (mix32(s) & mask));
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y;
  }
  if (acc == 12345.678f) sink[0] = acc;
}

__global__ void __launch_bounds__(256) k_peak_gather4(const float4* __restrict__ t, uint32_t mask, int iters,
                                                      float* __restrict__ sink) {
  uint32_t s = mix32(blockIdx.x * blockDim.x + threadIdx.x);
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      s = s * 1664525u + 1013904223u;
      v[u] = __ldg(t + (mix32(s) & mask));
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (acc == 12345.678f) sink[0] = acc;
}

__global__ void __launch_bounds__(256) k_peak_gather8(const float* __restrict__ t, uint32_t mask, int iters,
                                                      float* __restrict__ sink) {
  uint32_t s = mix32(blockIdx.x * blockDim.x + threadIdx.x + 31u);
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    float v[8][8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      s = s * 1664525u + 1013904223u;
      const float* p = t + 8 * size_t(mix32(s) & mask);
      asm volatile("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                   : "=f"(v[u][0]), "=f"(v[u][1]), "=f"(v[u][2]), "=f"(v[u][3]), "=f"(v[u][4]), "=f"(v[u][5]),
                     "=f"(v[u][6]), "=f"(v[u][7])
                   : "l"(p));
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc += v[u][e];
  }
  if (acc == 12345.678f) sink[0] = acc;
}

__global__ void __launch_bounds__(256) k_peak_red(float* __restrict__ t, uint32_t mask, int iters) {
  uint32_t s = mix32(blockIdx.x * blockDim.x + threadIdx.x + 777u);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      s = s * 1664525u + 1013904223u;
      atomicAdd(reinterpret_cast<float2*>(t) + (mix32(s) & mask), make_float2(1e-7f, 1e-7f));
    }
  }
}

__global__ void __launch_bounds__(256) k_peak_red4(float* __restrict__ t, uint32_t mask, int iters) {
  uint32_t s = mix32(blockIdx.x * blockDim.x + threadIdx.x + 777u);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      s = s * 1664525u + 1013904223u;
      atomicAdd(reinterpret_cast<float4*>(t) + (mix32(s) & mask), make_float4(1e-7f, 1e-7f, 1e-7f, 1e-7f));
    }
  }
}

__global__ void __launch_bounds__(256) k_peak_ffma(int iters, float* __restrict__ sink) {
  float a[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) a[u] = float(threadIdx.x + u);
  const float b = 1.0000001f, c = 1e-7f;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = fmaf(a[u], b, c);
  float r = 0.f;
#pragma unroll
  for (int u = 0; u < 8; ++u) r += a[u];
  if (r == 12345.678f) sink[0] = r;
}

__global__ void __launch_bounds__(256) k_peak_dfma(int iters, float* __restrict__ sink) {
  double a[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) a[u] = double(threadIdx.x + u);
  const double b = 1.0000000001, c = 1e-12;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = fma(a[u], b, c);
  double r = 0.0;
#pragma unroll
  for (int u = 0; u < 8; ++u) r += a[u];
  if (r == 12345.678) sink[0] = float(r);
}

__global__ void __launch_bounds__(128) k_peak_tf32(int iters) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  float* A = reinterpret_cast<float*>(sm);  // [128][8] CM
  float* B = A + 128 * 8;                   // [256][8] CM
  for (int e = threadIdx.x; e < (128 + 256) * 8; e += blockDim.x) A[e] = 1e-3f * float(e & 7);
  if (threadIdx.x < 32) umma::tmem_alloc(&slot, 256);
  if (threadIdx.x == 0) {
    umma::mbar_init(&bar, 1);
    umma::fence_mbar_init();
  }
  umma::fence_async_smem();
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = umma::idesc_tf32(128, 256, false, false);
    const uint64_t da = umma::desc_kmajor(umma::smem_u32(A), 128, 0);
    const uint64_t db = umma::desc_kmajor(umma::smem_u32(B), 256, 0);
    for (int it = 0; it < iters; ++it) umma::mma_tf32(tm, da, db, idesc, it > 0);
    umma::commit(&bar);
  }
  umma::mbar_wait(&bar, 0);
  umma::fence_after_sync();
  umma::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) umma::tmem_dealloc(tm, 256);
}

__global__ void __launch_bounds__(128) k_peak_bf16(int iters, int M, int N, int nacc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  unsigned char* A = sm;                  // [128][16] bf16 CM
  unsigned char* B = sm + 128 * 16 * 2;   // [256][16] bf16 CM
  for (int e = threadIdx.x; e < (128 + 256) * 16 * 2 / 4; e += blockDim.x) reinterpret_cast<uint32_t*>(sm)[e] = 0x3c003c00u;
  if (threadIdx.x < 32) umma::tmem_alloc(&slot, 256);
  if (threadIdx.x == 0) {
    umma::mbar_init(&bar, 1);
    umma::fence_mbar_init();
  }
  umma::fence_async_smem();
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = umma::idesc_bf16(M, N, false, false);
    const uint64_t da = umma::desc_kmajor(umma::smem_u32(A), M, 0);
    const uint64_t db = umma::desc_kmajor(umma::smem_u32(B), N, 0);
    if (nacc == 1) {
      umma::mma_bf16(tm, da, db, idesc, 0u);
      for (int it = 1; it < iters; it += 16)  // unrolled: the issue loop must not be the bound
#pragma unroll
        for (int u = 0; u < 16; ++u) umma::mma_bf16(tm, da, db, idesc, 1u);
    } else {
      for (int it = 0; it < iters; it += 16)
#pragma unroll
        for (int u = 0; u < 16; ++u) umma::mma_bf16(tm + 64 * (u & 3), da, db, idesc, it > 0 || u >= 4);
    }
    umma::commit(&bar);
  }
  umma::mbar_wait(&bar, 0);
  umma::fence_after_sync();
  umma::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) umma::tmem_dealloc(tm, 256);
}

__global__ void __launch_bounds__(256) k_peak_shfl(int iters, float* __restrict__ sink) {
  float v[4] = {float(threadIdx.x), 1.f, 2.f, 3.f};
  const int lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] += __shfl_sync(0xffffffffu, v[u], (lane + it + u) & 31);
  if (v[0] + v[1] + v[2] + v[3] == 12345.678f) sink[0] = v[0];
}

__global__ void __launch_bounds__(256) k_peak_atoms(int iters, float* __restrict__ sink) {
  __shared__ float s[8][32 * 17];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int e = lane; e < 32 * 17; e += 32) s[warp][e] = 0.f;
  __syncwarp();
  float* base = s[warp];
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int u = 0; u < 16; ++u) atomicAdd(base + lane * 17 + ((u + it) & 15), 1.f);
  __syncwarp();
  if (base[lane] == 12345.f) sink[0] = base[lane];
}

}  // namespace apmg

using namespace apmg;

extern "C" int apmg_peak_probe(int32_t kind, void* table, int64_t table_bytes, int32_t iters, double* work,
                               void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int sms = num_sms();
  float* sink = static_cast<float*>(table);
  switch (kind) {
    case 0:
    case 1: {
      APMG_ARG_CHECK(table && table_bytes >= 16 && (table_bytes & (table_bytes - 1)) == 0,
                     "table_bytes must be a power of two");
      const uint32_t mask = uint32_t(table_bytes / 8 - 1);
      const int grid = sms * 8, block = 256;
      if (kind == 0) {
        APMG_LAUNCH("peak_gather", k_peak_gather, grid, block, 0, st, static_cast<const float2*>(table), mask, iters,
                    sink);
        *work = double(grid) * block * iters * 8 * 8;
      } else {
        APMG_LAUNCH("peak_red", k_peak_red, grid, block, 0, st, static_cast<float*>(table), mask, iters);
        *work = double(grid) * block * iters * 8;
      }
      return APMG_OK;
    }
    case 2:
      APMG_LAUNCH("peak_ffma", k_peak_ffma, sms * 8, 256, 0, st, iters, sink);
      *work = double(sms) * 8 * 256 * iters * 8 * 2;
      return APMG_OK;
    case 3:
      APMG_LAUNCH("peak_dfma", k_peak_dfma, sms * 8, 256, 0, st, iters, sink);
      *work = double(sms) * 8 * 256 * iters * 8 * 2;
      return APMG_OK;
    case 4: {
      const int smem = (128 + 256) * 8 * 4;
      APMG_LAUNCH("peak_tf32", k_peak_tf32, sms, 128, smem, st, iters);
      *work = double(sms) * iters * 2.0 * 128 * 256 * 8;
      return APMG_OK;
    }
    case 5:
      APMG_LAUNCH("peak_shfl", k_peak_shfl, sms * 8, 256, 0, st, iters, sink);
      *work = double(sms) * 8 * 8 * iters * 4;  // warp-level shuffle instructions
      return APMG_OK;
    case 7: {
      APMG_ARG_CHECK(table && table_bytes >= 16 && (table_bytes & (table_bytes - 1)) == 0,
                     "table_bytes must be a power of two");
      const int grid = sms * 8, block = 256;
      APMG_LAUNCH("peak_gather4", k_peak_gather4, grid, block, 0, st, static_cast<const float4*>(table),
                  uint32_t(table_bytes / 16 - 1), iters, sink);
      *work = double(grid) * block * iters * 8 * 16;
      return APMG_OK;
    }
    case 10: {
      APMG_ARG_CHECK(table && table_bytes >= 32 && (table_bytes & (table_bytes - 1)) == 0,
                     "table_bytes must be a power of two");
      const int grid = sms * 8, block = 256;
      APMG_LAUNCH("peak_gather8", k_peak_gather8, grid, block, 0, st, static_cast<const float*>(table),
                  uint32_t(table_bytes / 32 - 1), iters, sink);
      *work = double(grid) * block * iters * 8 * 32;
      return APMG_OK;
    }
    case 8: {
      APMG_ARG_CHECK(table && table_bytes >= 16 && (table_bytes & (table_bytes - 1)) == 0,
                     "table_bytes must be a power of two");
      const int grid = sms * 8, block = 256;
      APMG_LAUNCH("peak_red4", k_peak_red4, grid, block, 0, st, static_cast<float*>(table),
                  uint32_t(table_bytes / 16 - 1), iters);
      *work = double(grid) * block * iters * 8;
      return APMG_OK;
    }
    case 9: {
      // table_bytes: N (16..256) + 1000 for M = 64 (else 128); 1 = N 64, 4 accumulators
      const int nacc = table_bytes == 1 ? 4 : 1;
      const int N = table_bytes == 1 ? 64 : int(table_bytes % 1000), M = table_bytes >= 1000 ? 64 : 128;
      const int smem = (128 + 256) * 16 * 2;
      APMG_LAUNCH("peak_bf16", k_peak_bf16, sms, 128, smem, st, iters, M, N, nacc);
      *work = double(sms) * iters * 2.0 * M * N * 16;
      return APMG_OK;
    }
    case 6:
      APMG_LAUNCH("peak_atoms", k_peak_atoms, sms * 8, 256, 0, st, iters, sink);
      *work = double(sms) * 8 * 8 * iters * 16;  // warp-level atomic instructions
      return APMG_OK;
    default:
      set_error("unknown probe kind %d", kind);
      return APMG_E_ARG;
  }
}
