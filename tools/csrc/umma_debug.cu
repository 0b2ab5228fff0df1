// Self-test of the tcgen05 operand/descriptor conventions used by the fused MLP
// (umma.cuh): one CTA runs one small GEMM from row-major f32 inputs staged in the
// CM layout, optionally with the 3xTF32 split, and writes D row-major.
//   cfg 0: D[64][N]  = A[64][K]  . B[N][K]^T   (A K-major, B K-major)   e.g. z1 = F W1^T
//   cfg 1: D[64][N]  = A[64][K]  . B[K][N]     (A K-major, B MN-major)  e.g. gF = dz1 W1
//   cfg 2: D[128][N] = A[K][128]^T . B[K][N]   (A MN-major, B MN-major) e.g. dW1^T = F^T dz1
//   cfg 3: D[128][N] = A[128][K] . B[N][K]^T   (M = 128, K-major both)
//   cfg 4: D[128][N] = A[128][K] . B[N][K]^T   (A from tensor memory, cols 128.., B K-major)
#include "common.cuh"
#include "umma.cuh"

namespace apmg {

__global__ void __launch_bounds__(128) k_umma_debug(int cfg_flags, int K, int N, int split3, const float* __restrict__ A,
                                                    const float* __restrict__ B, float* __restrict__ D) {
  const int cfg = cfg_flags & 15;
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tbase;
  const int M = (cfg >= 2) ? 128 : 64;
  // A rows x cols and B rows x cols as stored (row-major inputs)
  const int a_rows = (cfg == 2) ? K : M, a_cols = (cfg == 2) ? 128 : K;
  const bool bk = (cfg == 0 || cfg == 3 || cfg == 4);
  const int b_rows = bk ? N : K, b_cols = bk ? K : N;
  float *Ah, *Al, *Bh, *Bl;
  if (cfg_flags & 256) {  // B first in smem
    Bh = reinterpret_cast<float*>(sm);
    Bl = Bh + b_rows * b_cols;
    Ah = Bl + b_rows * b_cols;
    Al = Ah + a_rows * a_cols;
  } else {
    Ah = reinterpret_cast<float*>(sm);
    Al = Ah + a_rows * a_cols;
    Bh = Al + a_rows * a_cols;
    Bl = Bh + b_rows * b_cols;
  }
  // flag 8192: "RG" layout (K chunks of one 8-row group adjacent): offset = (r/8)*SR + (c/4)*128 + (r%8)*16 + (c%4)*4
  const bool rg = cfg_flags & 8192;
  auto rg_off = [](int r, int c, int cols) {
    return uint32_t((r >> 3) * ((cols / 4) * 128) + (c >> 2) * 128 + (r & 7) * 16 + (c & 3) * 4);
  };
  // flag 131072: MN-major operands (cfg 1 B, cfg 2 A/B) use the CUTLASS-canonical arrangement:
  // rows = K, cols = MN: offset = (r/8)*((cols/4)*128) + (c/4)*128 + (r%8)*16 + (c%4)*4  == rg_off
  const bool mnc = cfg_flags & 131072;
  for (int e = threadIdx.x; e < a_rows * a_cols; e += blockDim.x) {
    const int r = e / a_cols, c = e % a_cols;
    const float x = (cfg_flags & 64) ? 0.f : A[e];
    float hi, lo;
    umma::split_tf32(x, hi, lo);
    const bool amn = (cfg == 2);
    const uint32_t off = ((rg || (mnc && amn)) ? rg_off(r, c, a_cols) : umma::cm_offset(r, c, a_rows)) / 4;
    Ah[off] = split3 ? hi : x;
    Al[off] = lo;
  }
  for (int e = threadIdx.x; e < b_rows * b_cols; e += blockDim.x) {
    const int r = e / b_cols, c = e % b_cols;
    const float x = (cfg_flags & 32) ? 0.f : B[e];
    float hi, lo;
    umma::split_tf32(x, hi, lo);
    const bool bmn = (cfg == 1 || cfg == 2);
    const uint32_t off = ((rg || (mnc && bmn)) ? rg_off(r, c, b_cols) : umma::cm_offset(r, c, b_rows)) / 4;
    Bh[off] = split3 ? hi : x;
    Bl[off] = lo;
  }
  if (cfg_flags & 32768) {  // dump the staged A_hi buffer (raw smem order) and return
    __syncthreads();
    for (int e = threadIdx.x; e < a_rows * a_cols; e += blockDim.x) D[e] = Ah[e];
    return;
  }
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
  if (cfg_flags & (1024 | 2048)) {  // pre-fill TMEM columns [0, 64) with 0 or lane*1000+col
    const int w = threadIdx.x >> 5, t = threadIdx.x & 31;
    for (int c0 = 0; c0 < 64; c0 += 16) {
      uint32_t r[16];
      for (int i = 0; i < 16; ++i)
        r[i] = __float_as_uint((cfg_flags & 2048) ? float((32 * w + t) * 1000 + c0 + i) : 0.f);
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
              umma::taddr(tb, 32 * w, c0)),
          "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
          "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
  }
  if (cfg == 4) {  // A (hi at column 128, lo at 128 + K) into tensor memory, lane = row
    const int w = threadIdx.x >> 5, t = threadIdx.x & 31, row = 32 * w + t;
    for (int c0 = 0; c0 < K; c0 += 16) {
      uint32_t rh[16], rl[16];
      for (int i = 0; i < 16; ++i) {
        const float x = (c0 + i < K) ? A[row * K + c0 + i] : 0.f;
        float hi, lo;
        umma::split_tf32(x, hi, lo);
        rh[i] = __float_as_uint(split3 ? hi : x);
        rl[i] = __float_as_uint(lo);
      }
      umma::tmem_st16(umma::taddr(tb, 32 * w, 128 + c0), rh);
      umma::tmem_st16(umma::taddr(tb, 32 * w, 128 + K + c0), rl);
    }
    umma::tmem_st_wait();
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
  }
  if (threadIdx.x == 0 && cfg == 4) {
    const uint32_t idesc = umma::idesc_tf32(128, N, false, false);
    const uint32_t sBh = umma::smem_u32(Bh), sBl = umma::smem_u32(Bl);
    for (int kk = 0; kk < K / 8; ++kk) {
      const uint64_t bh = umma::desc_kmajor(sBh, b_rows, kk), bl = umma::desc_kmajor(sBl, b_rows, kk);
      umma::mma_tf32_ts(tb, umma::taddr(tb, 0, 128 + 8 * kk), bh, idesc, kk > 0);
      if (split3) {
        umma::mma_tf32_ts(tb, umma::taddr(tb, 0, 128 + 8 * kk), bl, idesc, 1);
        umma::mma_tf32_ts(tb, umma::taddr(tb, 0, 128 + K + 8 * kk), bh, idesc, 1);
      }
    }
    umma::commit(&mbar);
  } else if (threadIdx.x == 0) {
    const bool a_mn = (cfg == 2), b_mn = (cfg == 1 || cfg == 2);
    const uint32_t idesc = umma::idesc_tf32(M, N, a_mn, b_mn);
    const uint32_t sAh = umma::smem_u32(Ah), sAl = umma::smem_u32(Al), sBh = umma::smem_u32(Bh),
                   sBl = umma::smem_u32(Bl);
    uint32_t acc = 0;
    if (cfg_flags & 16) printf("umma_debug: sAh=%u sAl=%u sBh=%u sBl=%u idesc=%08x descA0=%016llx descB0=%016llx tmem=%08x\n",
                         sAh, sAl, sBh, sBl, idesc,
                         (unsigned long long)(a_mn ? umma::desc_mnmajor(sAh, a_rows, 0) : umma::desc_kmajor(sAh, a_rows, 0)),
                         (unsigned long long)(b_mn ? umma::desc_mnmajor(sBh, b_rows, 0) : umma::desc_kmajor(sBh, b_rows, 0)), tb);
    for (int kk = 0; kk < K / 8; ++kk) {
      const bool swp = cfg_flags & 16384;
      auto kdesc = [&](uint32_t base, int rows, int cols) {
        uint32_t start, lbo, sbo;
        if (rg) {
          start = base + uint32_t(kk) * 256u;
          lbo = 128u;
          sbo = uint32_t((cols / 4) * 128);
        } else {
          start = base + uint32_t(kk) * 2u * uint32_t(rows * 16);
          lbo = uint32_t(rows * 16);
          sbo = 128u;
        }
        return swp ? umma::smem_desc(start, sbo, lbo) : umma::smem_desc(start, lbo, sbo);
      };
      auto mdesc = [&](uint32_t base, int rows, int cols) {
        if (mnc) return umma::smem_desc(base + uint32_t(kk) * uint32_t((cols / 4) * 128), uint32_t((cols / 4) * 128), 128u);
        if (cfg_flags & 65536) return umma::smem_desc(base + uint32_t(kk) * 128u, uint32_t(rows * 16), 128u);
        return umma::desc_mnmajor(base, rows, kk);
      };
      auto da = [&](uint32_t base) { return a_mn ? mdesc(base, a_rows, a_cols) : kdesc(base, a_rows, a_cols); };
      auto db = [&](uint32_t base) { return b_mn ? mdesc(base, b_rows, b_cols) : kdesc(base, b_rows, b_cols); };
      if (cfg_flags & 128)
        umma::mma_tf32(tb, db(sBh), da(sAh), idesc, acc);
      else if (cfg_flags & 4096)
        umma::mma_tf32_mask(tb, da(sAh), db(sBh), idesc, acc);
      else
        umma::mma_tf32(tb, da(sAh), db(sBh), idesc, acc);
      acc = 1;
      if (split3) {
        umma::mma_tf32(tb, da(sAh), db(sBl), idesc, 1);
        umma::mma_tf32(tb, da(sAl), db(sBh), idesc, 1);
      }
    }
    umma::commit(&mbar);
  }
  umma::mbar_wait(&mbar, 0);
  umma::fence_after_sync();
  const int w = threadIdx.x >> 5, t = threadIdx.x & 31;
  if (cfg_flags & 512) {  // TMEM store/load round trip: value = lane*1000 + column
    for (int c0 = 0; c0 < N; c0 += 16) {
      uint32_t r[16];
      for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(float((32 * w + t) * 1000 + c0 + i));
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
              umma::taddr(tb, 32 * w, c0)),
          "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
          "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
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

extern "C" int apmg_debug_umma_gemm(int32_t cfg, int32_t K, int32_t N, int32_t split3, const float* A, const float* B,
                                    float* D, void* stream) {
  APMG_ARG_CHECK((cfg & 15) <= 4, "cfg 0..4 (+16: print descriptors)");
  APMG_ARG_CHECK((cfg & 15) != 4 || (K <= 64 && N <= 128), "cfg 4: K <= 64, N <= 128");
  APMG_ARG_CHECK(K % 8 == 0 && K >= 8 && K <= 128, "K multiple of 8 in [8,128]");
  APMG_ARG_CHECK(N % 16 == 0 && N >= 16 && N <= 256, "N multiple of 16 in [16,256]");
  const int M = (cfg & 15) >= 2 ? 128 : 64;
  const size_t smem = sizeof(float) * 2 * (size_t(M) * K + size_t(K) * N);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  APMG_CUDA_TRY(cudaFuncSetAttribute(k_umma_debug, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  APMG_LAUNCH("umma_debug", k_umma_debug, 1, 128, smem, st, cfg, K, N, split3, A, B, D);
  return APMG_OK;
}
