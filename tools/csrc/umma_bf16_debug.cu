// Self-test of the 16-bit tcgen05 operand conventions (umma.cuh, kind::f16 with BF16
// inputs): one CTA computes D[M][N] = A . B from row-major f32 inputs split into bf16x3 and
// staged in the 16-bit CM layout, with each operand K-major or MN-major.
//   mode bit 0: B MN-major (stored [K][N]) instead of K-major ([N][K])
//   mode bit 1: A MN-major (stored [K][M]) instead of K-major ([M][K])
//   split3: 6 products (hh, hm, mh, hl, lh, mm) instead of 1 (hh)
#include "common.cuh"
#include "umma.cuh"

namespace apmg {

__global__ void __launch_bounds__(128) k_umma_bf16(int mode, int M, int K, int N, int split3,
                                                   const float* __restrict__ A, const float* __restrict__ B,
                                                   float* __restrict__ D) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tbase;
  const bool a_mn = mode & 2, b_mn = mode & 1;
  // three splits of A then of B, each one CM buffer
  const int a_rows = a_mn ? K : M, a_cols = a_mn ? M : K;
  const int b_rows = b_mn ? K : N, b_cols = b_mn ? N : K;
  const uint32_t a_bytes = uint32_t(M) * K * 2, b_bytes = uint32_t(N) * K * 2;
  unsigned char* As[3] = {sm, sm + a_bytes, sm + 2 * a_bytes};
  unsigned char* Bs[3] = {sm + 3 * a_bytes, sm + 3 * a_bytes + b_bytes, sm + 3 * a_bytes + 2 * b_bytes};
  for (int e = threadIdx.x; e < M * K; e += blockDim.x) {
    const int i = e / K, k = e % K;  // A[i][k]
    __nv_bfloat16 h, m, l;
    umma::split_bf16x3(A[e], h, m, l);
    const uint32_t o = a_mn ? umma::cm16_offset(k, i, a_rows) : umma::cm16_offset(i, k, a_rows);
    *reinterpret_cast<__nv_bfloat16*>(As[0] + o) = h;
    *reinterpret_cast<__nv_bfloat16*>(As[1] + o) = m;
    *reinterpret_cast<__nv_bfloat16*>(As[2] + o) = l;
  }
  for (int e = threadIdx.x; e < K * N; e += blockDim.x) {
    const int k = e / N, j = e % N;  // B[k][j]
    __nv_bfloat16 h, m, l;
    umma::split_bf16x3(B[e], h, m, l);
    const uint32_t o = b_mn ? umma::cm16_offset(k, j, b_rows) : umma::cm16_offset(j, k, b_rows);
    *reinterpret_cast<__nv_bfloat16*>(Bs[0] + o) = h;
    *reinterpret_cast<__nv_bfloat16*>(Bs[1] + o) = m;
    *reinterpret_cast<__nv_bfloat16*>(Bs[2] + o) = l;
  }
  (void)a_cols;
  (void)b_cols;
  if (threadIdx.x < 32) umma::tmem_alloc(&tbase, 256);
  if (threadIdx.x == 0) {
    umma::mbar_init(&mbar, 1);
    umma::fence_mbar_init();
  }
  umma::fence_async_smem();
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tb = tbase;
  if (threadIdx.x == 0) {
    const uint32_t idesc = umma::idesc_bf16(M, N, a_mn, b_mn);
    auto da = [&](int s, int kk) {
      const uint32_t b = umma::smem_u32(As[s]);
      return a_mn ? umma::desc_mnmajor16(b, a_rows, kk) : umma::desc_kmajor(b, a_rows, kk);
    };
    auto db = [&](int s, int kk) {
      const uint32_t b = umma::smem_u32(Bs[s]);
      return b_mn ? umma::desc_mnmajor16(b, b_rows, kk) : umma::desc_kmajor(b, b_rows, kk);
    };
    const int pa[6] = {0, 0, 1, 0, 2, 1}, pb[6] = {0, 1, 0, 2, 0, 1};
    for (int kk = 0; kk < K / 16; ++kk)
      for (int q = 0; q < (split3 ? 6 : 1); ++q)
        umma::mma_bf16(tb, da(pa[q], kk), db(pb[q], kk), idesc, (kk > 0 || q > 0) ? 1u : 0u);
    umma::commit(&mbar);
  }
  umma::mbar_wait(&mbar, 0);
  umma::fence_after_sync();
  const int w = threadIdx.x >> 5, t = threadIdx.x & 31;
  int row = -1;
  if (M == 128) row = 32 * w + t;
  else if (t < 16) row = 16 * w + t;
  for (int c0 = 0; c0 < N; c0 += 16) {
    float v[16];
    umma::tmem_ld16(umma::taddr(tb, 32 * w, c0), v);
    if (row >= 0)
      for (int i = 0; i < 16; ++i) D[row * N + c0 + i] = v[i];
  }
  umma::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) umma::tmem_dealloc(tb, 256);
}

}  // namespace apmg

using namespace apmg;

extern "C" int apmg_debug_umma_bf16(int32_t mode, int32_t M, int32_t K, int32_t N, int32_t split3, const float* A,
                                    const float* B, float* D, void* stream) {
  APMG_ARG_CHECK(mode >= 0 && mode <= 3, "mode 0..3");
  APMG_ARG_CHECK(M == 64 || M == 128, "M 64 or 128");
  APMG_ARG_CHECK(K % 16 == 0 && K >= 16 && K <= 128, "K multiple of 16 in [16,128]");
  APMG_ARG_CHECK(N % 16 == 0 && N >= 16 && N <= 256, "N multiple of 16 in [16,256]");
  const size_t smem = size_t(3) * 2 * (size_t(M) * K + size_t(K) * N);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  APMG_CUDA_TRY(cudaFuncSetAttribute(k_umma_bf16, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  APMG_LAUNCH("umma_bf16_debug", k_umma_bf16, 1, 128, smem, st, mode, M, K, N, split3, A, B, D);
  return APMG_OK;
}
