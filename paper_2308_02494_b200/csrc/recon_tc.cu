// Fused reconstruction step (optim.py:102-155) for the flagship shape
// (float32, 64 grids x 2 channels -> 128 features, 64 hidden), tensor-core MLP.
//
// One persistent CTA (16 warps) per SM; a 64-point tile per loop iteration:
//   encode      (point, grid) pairs -> features F, split hi/lo (3xTF32), CM layout in smem;
//               the cell terms of each pair stay in the owning thread's TMEM slots
//   z1 = F W1^T   tcgen05.mma kind::tf32 (A, B from smem), M=64 N=64 K=128, 3 products
//   h1 = relu     epilogue -> h1 hi/lo (smem), sign bitmap of h1
//   z2 = h1 W2^T  tcgen05.mma, M=64 N=64 K=64, 3 products
//   head/loss     epilogue: out = h2 w3 * span + vmin, residual, sq error, g = dL/dout,
//                 mask[p][j] = [z2 > 0] (exact 0/1 operand)
//   dz1^T = V mask^T       tcgen05.mma with A = V = (w3 o W2)^T resident in TMEM (M=128,
//                 rows 64..127 repeat 0..63), B = mask; dz1[p][i] = g[p] dz1^T[i][p] [h1 > 0].
//                 (g_z2 = g w3^T [z2>0] is rank one per row, optim.py:143-145, so its
//                 product with W2 needs only the split of V: 2 products, exact mask.)
//   gF^T = W1^T dz1^T      tcgen05.mma, A = W1^T resident in TMEM (M=128), B = dz1 hi/lo
//   dW2 += dz2^T h1, dW1 += dz1^T F   register-fragment MMAs (mma.sync m16n8k8 tf32,
//                 round-to-nearest operands), overlapped with the tcgen05 products
//   scatter       gF -> channel-last grid gradients (warp-aggregated float2 RED)
// The next tile's encode follows each thread's scatter without a barrier.
//
// Shared memory (215 KB): W1 hi/lo | W2 hi/lo | F hi/lo | h1 hi/lo -> dz1 hi/lo -> gF |
// mask | small.  Tensor memory (512 columns): acc A (z1, then dz1^T) | acc B (z2, then gF^T)
// | per-thread cell cache | V hi/lo | W1^T hi/lo.
#include "kernels.cuh"
#include "umma.cuh"

namespace apmg {
namespace tc {

constexpr int P = 64;     // points per tile (M of the forward tcgen05 products)
constexpr int NW = 16;    // warps per CTA
constexpr int NT = 32 * NW;
constexpr int WQ = NW / 4;    // warps sharing one TMEM lane quarter
constexpr int EPC = 64 / WQ;  // accumulator columns per warp in the epilogues (16)
constexpr int GPW = 64 / NW;  // grids per warp in encode / scatter (4)
constexpr int NT64 = 32 / NW;   // 16x8 n-tiles per warp of a 64x64 mma.sync product (2)
constexpr int NT128 = 64 / NW;  // 16x8 n-tiles per warp of a 64x128 product (4)
constexpr int FE = 128;         // features
constexpr int HID = 64;
static_assert(EPC == 16 && GPW % 2 == 0, "epilogue / cache mappings assume 16 warps");

// shared memory map (bytes)
constexpr uint32_t OFF_W1H = 0;
constexpr uint32_t OFF_W1L = OFF_W1H + 64 * 128 * 4;
constexpr uint32_t OFF_W2H = OFF_W1L + 64 * 128 * 4;
constexpr uint32_t OFF_W2L = OFF_W2H + 64 * 64 * 4;
constexpr uint32_t OFF_FH = OFF_W2L + 64 * 64 * 4;
constexpr uint32_t OFF_FL = OFF_FH + P * FE * 4;
constexpr uint32_t OFF_H1H = OFF_FL + P * FE * 4;    // h1 hi -> dz1 hi -> gF (first half)
constexpr uint32_t OFF_H1L = OFF_H1H + P * HID * 4;  // h1 lo -> dz1 lo -> gF (second half)
constexpr uint32_t OFF_MASK = OFF_H1L + P * HID * 4;
constexpr uint32_t OFF_X = OFF_MASK + P * HID * 4;   // [2][P][3] coordinates (double buffered)
constexpr uint32_t OFF_T = OFF_X + 2 * P * 3 * 4;    // [2][P] targets
constexpr uint32_t OFF_G = OFF_T + 2 * P * 4;        // [P] dL/dout
constexpr uint32_t OFF_HEAD = OFF_G + P * 4;         // [WQ][P] head partial sums
constexpr uint32_t OFF_DW3 = OFF_HEAD + WQ * P * 4;  // [64]
constexpr uint32_t OFF_RED = OFF_DW3 + HID * 4;      // [32] doubles
constexpr uint32_t OFF_BAR = OFF_RED + 32 * 8;
constexpr uint32_t OFF_TM = OFF_BAR + 8;
constexpr uint32_t OFF_TF = OFF_TM + 8;              // [64][12] transforms (f32)
constexpr uint32_t OFF_W3 = OFF_TF + 64 * 12 * 4;    // [64]
constexpr uint32_t OFF_M1 = OFF_W3 + 64 * 4;         // [64 i][4] u16: bit p%16 of word p/16 = [h1[p][i] > 0]
constexpr uint32_t SMEM_BYTES = OFF_M1 + 64 * 4 * 2;
static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");

// tensor memory columns
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t TC_ACC_A = 0, TC_ACC_B = 64, TC_CACHE = 128, TC_VH = 256, TC_VL = 320, TC_W1TH = 384,
                   TC_W1TL = 448;

// per-phase clock stamps of CTA 0 / thread 0 for the first 16 tiles (APMG_TC_SKIP & 64)
__device__ long long g_tc_stamp[16][12];
#define TC_STAMP(k)                                                                 \
  do {                                                                              \
    if ((a.skip & 64) && blockIdx.x == 0 && tid == 0 && it < 16) g_tc_stamp[it][k] = clock64(); \
  } while (0)

__device__ __forceinline__ float* fptr(unsigned char* sm, uint32_t off) { return reinterpret_cast<float*>(sm + off); }

// float index of column c in a 64-row CM buffer (row part: (r/8)*32 + (r%8)*4)
__device__ __forceinline__ uint32_t cm_col(int c) { return uint32_t((c >> 2) * 256 + (c & 3)); }
__device__ __forceinline__ uint32_t cm64(int r, int c) { return umma::cm_offset(r, c, 64) >> 2; }

// gF [P][128] in the 32 KB h1 region: row stride 128, 8-byte granules XOR-swizzled by row so
// that both the column-per-lane epilogue writes and the row-per-lane float2 scatter reads
// are conflict-free
__device__ __forceinline__ int gf_idx(int p, int k) { return p * 128 + (k ^ ((p & 15) << 1)); }

__device__ __forceinline__ uint32_t tf32_bits(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ void mma_tf32_16x8x8(float* d, const uint32_t* a, const uint32_t* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

struct Args {
  ModelDev<float> md;
  int64_t n;
  const float* coords;
  const float* targets;
  float* sq;
  float* dgrid;
  float* part_dw;
  double* part_loss;
  const TrainCtl* ctl;
  int aggregate;  // warp-aggregated scatter (APMG_SCATTER_AGG=0 disables, for A/B)
  int skip;       // timing breakdown only (APMG_TC_SKIP): 1 scatter, 2 register MMAs, 4 gathers
};

// Grid-gradient scatter of one (2 grids x 2 points) group of a tile: thread (warp, lane)
// owns points lane, lane + 32 and grids warp + NW*j, exactly the items it encoded; their
// cell terms come back from its TMEM cache, their feature gradients from gF.
__device__ __forceinline__ void scatter_group(const ModelDev<float>& md, const Args& a, const float* GF,
                                              uint32_t tmem_cache, int jq, int cnt, int warp, int lane) {
  if (a.skip & 1) return;
  uint32_t cache[16];
  umma::tmem_ld16u(tmem_cache + 16 * jq, cache);
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int j = 2 * jq + (u >> 1), h = u & 1;
    const int m = warp + NW * j, p = lane + 32 * h;
    const int vbase = int(cache[4 * u]);
    const bool valid = vbase >= 0 && p < cnt;
    float2 g = make_float2(0.f, 0.f);
    if (valid) g = *reinterpret_cast<const float2*>(GF + gf_idx(p, 2 * m));
    if (a.aggregate)
      scatter_vertex_warp_agg(md, a.dgrid, valid, vbase, __uint_as_float(cache[4 * u + 1]),
                              __uint_as_float(cache[4 * u + 2]), __uint_as_float(cache[4 * u + 3]), g.x, g.y);
    else if (valid)
      scatter_vertex_f32(md, a.dgrid, vbase, __uint_as_float(cache[4 * u + 1]), __uint_as_float(cache[4 * u + 2]),
                         __uint_as_float(cache[4 * u + 3]), g.x, g.y);
  }
}

__device__ __forceinline__ void load_tile(const Args& a, int64_t tile, float* sX, float* sT, int tid) {
  if (tid < P) {
    const int64_t i = tile * P + tid;
    const bool ok = i < a.n;
    sX[3 * tid] = ok ? a.coords[3 * i] : 0.f;
    sX[3 * tid + 1] = ok ? a.coords[3 * i + 1] : 0.f;
    sX[3 * tid + 2] = ok ? a.coords[3 * i + 2] : 0.f;
    sT[tid] = ok ? a.targets[i] : 0.f;
  }
}

__global__ void __launch_bounds__(NT, 1) k_recon_tc(Args a) {
  extern __shared__ __align__(1024) unsigned char sm[];
  if (a.ctl && a.ctl->skip) return;
  const ModelDev<float>& md = a.md;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const int quarter = warp & 3, wq = warp >> 2;  // TMEM lane quarter, index among its WQ warps
  float* W1h = fptr(sm, OFF_W1H);
  float* W1l = fptr(sm, OFF_W1L);
  float* W2h = fptr(sm, OFF_W2H);
  float* W2l = fptr(sm, OFF_W2L);
  float* Fh = fptr(sm, OFF_FH);
  float* Fl = fptr(sm, OFF_FL);
  float* H1h = fptr(sm, OFF_H1H);
  float* H1l = fptr(sm, OFF_H1L);
  float* DZ1h = H1h;  // dz1 replaces h1 once dW2 has consumed it
  float* DZ1l = H1l;
  float* GF = H1h;    // gF replaces dz1 once gF^T and dW1 have consumed it (32 KB)
  float* MASK = fptr(sm, OFF_MASK);
  float* sX = fptr(sm, OFF_X);
  float* sT = fptr(sm, OFF_T);
  float* sG = fptr(sm, OFF_G);
  float* sHead = fptr(sm, OFF_HEAD);
  float* sDW3 = fptr(sm, OFF_DW3);
  double* red = reinterpret_cast<double*>(sm + OFF_RED);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + OFF_BAR);
  uint32_t* tm_slot = reinterpret_cast<uint32_t*>(sm + OFF_TM);
  float* sTF = fptr(sm, OFF_TF);
  float* sW3 = fptr(sm, OFF_W3);
  uint16_t* sM1 = reinterpret_cast<uint16_t*>(sm + OFF_M1);

  // ---- stage weights (hi/lo, CM layout, rows = output unit) ----
  for (int e = tid; e < 64 * 128; e += NT) {
    const int r = e >> 7, c = e & 127;
    float hi, lo;
    umma::split_tf32(md.w1[e], hi, lo);
    const uint32_t o = umma::cm_offset(r, c, 64) >> 2;
    W1h[o] = hi;
    W1l[o] = lo;
  }
  for (int e = tid; e < 64 * 64; e += NT) {
    const int r = e >> 6, c = e & 63;
    float hi, lo;
    umma::split_tf32(md.w2[e], hi, lo);
    const uint32_t o = umma::cm_offset(r, c, 64) >> 2;
    W2h[o] = hi;
    W2l[o] = lo;
  }
  if (tid < HID) sDW3[tid] = 0.f;
  for (int e = tid; e < 64 * 12; e += NT) sTF[e] = md.tf[16 * (e / 12) + (e % 12)];
  if (tid < HID) sW3[tid] = md.w3[tid];
  if (warp == 0) umma::tmem_alloc(tm_slot, TMEM_COLS);
  if (tid == 0) {
    umma::mbar_init(bar, 1);
    umma::fence_mbar_init();
  }
  const int64_t tiles = ceil_div(a.n, P);
  load_tile(a, blockIdx.x, sX, sT, tid);
  umma::fence_async_smem();
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tmem = *tm_slot;
  const uint32_t lane_base = uint32_t(32 * quarter) << 16;
  const uint32_t TZ1 = tmem + TC_ACC_A, TZ2 = tmem + TC_ACC_B;
  // the WQ warps sharing a lane quarter use disjoint 8*GPW-column slices of the cache
  const uint32_t tmem_cache = tmem + TC_CACHE + 8 * GPW * wq + lane_base;

  // ---- resident A operands in TMEM (row = lane): V[i][j] = w3[j] W2[j][i] (rows 64-127
  // repeat rows 0-63, so all four lane quarters receive dz1^T) and W1^T[k][i] = W1[i][k];
  // warps 0-3 write V, warps 4-7 write W1^T ----
  if (warp < 8) {
    const int r = 32 * quarter + lane;
    const bool is_v = warp < 4;
#pragma unroll 1
    for (int c0 = 0; c0 < 64; c0 += 16) {
      uint32_t rh[16], rl[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        float x;
        if (is_v)
          x = __fmul_rn(md.w3[c0 + c], md.w2[(c0 + c) * HID + (r & (HID - 1))]);
        else
          x = md.w1[(c0 + c) * FE + r];
        float hi, lo;
        umma::split_tf32(x, hi, lo);
        rh[c] = __float_as_uint(hi);
        rl[c] = __float_as_uint(lo);
      }
      umma::tmem_st16(tmem + lane_base + (is_v ? TC_VH : TC_W1TH) + c0, rh);
      umma::tmem_st16(tmem + lane_base + (is_v ? TC_VL : TC_W1TL) + c0, rl);
    }
    umma::tmem_st_wait();
  }
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();

  const uint32_t sW1h = umma::smem_u32(W1h), sW1l = umma::smem_u32(W1l), sW2h = umma::smem_u32(W2h),
                 sW2l = umma::smem_u32(W2l), sFh = umma::smem_u32(Fh), sFl = umma::smem_u32(Fl),
                 sH1h = umma::smem_u32(H1h), sH1l = umma::smem_u32(H1l), sMask = umma::smem_u32(MASK);
  const uint32_t idesc64 = umma::idesc_tf32(64, 64, false, false);
  const uint32_t idesc128 = umma::idesc_tf32(128, 64, false, false);
  const float coef = __fmul_rn(float(2.0 / double(a.n)), md.span);

  // persistent weight-gradient accumulators (mma.sync fragments); warp w owns m-tile
  // mt = w / WQ (16 rows) and a contiguous run of 8-column n-tiles
  const int mt = warp / WQ, wn = warp % WQ;
  float acc1[NT128][4];  // dW1 [64 i][128 k]: n-tiles NT128*wn ..
  float acc2[NT64][4];   // dW2 [64 j][64 i]:  n-tiles NT64*wn ..
#pragma unroll
  for (int t = 0; t < NT128; ++t)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc1[t][e] = 0.f;
#pragma unroll
  for (int t = 0; t < NT64; ++t)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc2[t][e] = 0.f;
  float dw3_acc[EPC];
#pragma unroll
  for (int c = 0; c < EPC; ++c) dw3_acc[c] = 0.f;
  double loss = 0.0;
  uint32_t phase = 0;

  // M=64 accumulator epilogue mapping: row 16*q + t lives in lane 32*q + t (t < 16)
  const int ep_row = 16 * quarter + lane;  // valid when lane < 16
  const int ep_col0 = EPC * wq;            // the WQ warps of a quarter split the 64 columns

  // encode of one (2 grids x 2 points) group: lane -> point, warp -> grid; features split
  // hi/lo into F, cell terms cached in TMEM for the scatter
  auto encode_group = [&](const float* cX, int jq) {
    const float xa[2][3] = {{cX[3 * lane], cX[3 * lane + 1], cX[3 * lane + 2]},
                            {cX[3 * (lane + 32)], cX[3 * (lane + 32) + 1], cX[3 * (lane + 32) + 2]}};
    uint32_t cache[16];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = 2 * jq + (u >> 1), h = u & 1;
      const int m = warp + NW * j, p = lane + 32 * h;
      const float* tf = sTF + 12 * m;
      const float l0 = local_coord(xa[h][0], xa[h][1], xa[h][2], tf[0], tf[1], tf[2], tf[3]);
      const float l1 = local_coord(xa[h][0], xa[h][1], xa[h][2], tf[4], tf[5], tf[6], tf[7]);
      const float l2 = local_coord(xa[h][0], xa[h][1], xa[h][2], tf[8], tf[9], tf[10], tf[11]);
      const bool inside = (fabsf(l0) <= 1.f) && (fabsf(l1) <= 1.f) && (fabsf(l2) <= 1.f);
      int ix, iy, iz;
      double fxd, fyd, fzd;
      axis_term(l0, md.W, ix, fxd);
      axis_term(l1, md.H, iy, fyd);
      axis_term(l2, md.D, iz, fzd);
      const float fx = float(fxd), fy = float(fyd), fz = float(fzd);
      const int vbase = inside ? ((m * md.D + iz) * md.H + iy) * md.W + ix : -1;
      float f0 = 0.f, f1 = 0.f;
      if (inside && !(a.skip & 4)) interp_pair_f32(md.grid, md.W, md.H * md.W, vbase, fx, fy, fz, f0, f1);
      cache[4 * u] = uint32_t(vbase);
      cache[4 * u + 1] = __float_as_uint(fx);
      cache[4 * u + 2] = __float_as_uint(fy);
      cache[4 * u + 3] = __float_as_uint(fz);
      float hi0, lo0, hi1, lo1;
      umma::split_tf32(f0, hi0, lo0);
      umma::split_tf32(f1, hi1, lo1);
      const uint32_t o = umma::cm_offset(p, 2 * m, 64) >> 2;
      *reinterpret_cast<float2*>(Fh + o) = make_float2(hi0, hi1);
      *reinterpret_cast<float2*>(Fl + o) = make_float2(lo0, lo1);
    }
    umma::tmem_st16(tmem_cache + 16 * jq, cache);
  };
  // z1 = F W1^T (3xTF32) over K-steps [k0, k1), committed when `last`
  auto issue_z1 = [&](int k0, int k1, bool last) {
    if (tid != 0) return;
    umma::fence_after_sync();
    for (int kk = k0; kk < k1; ++kk) {
      const uint64_t fh = umma::desc_kmajor(sFh, 64, kk), fl = umma::desc_kmajor(sFl, 64, kk);
      const uint64_t wh = umma::desc_kmajor(sW1h, 64, kk), wl = umma::desc_kmajor(sW1l, 64, kk);
      umma::mma_tf32(TZ1, fh, wh, idesc64, kk > 0);
      umma::mma_tf32(TZ1, fh, wl, idesc64, 1);
      umma::mma_tf32(TZ1, fl, wh, idesc64, 1);
    }
    if (last) umma::commit(bar);
  };
  // Encode of tile t+1 is interleaved group by group with the scatter of tile t in every
  // thread (scatter: shuffle-crossbar bound; encode: L2-latency bound), and the first half
  // of z1 (features of grids 0-31) starts as soon as group 0 is written everywhere.
  // `scatter_cnt` < 0: no scatter (first tile).
  auto encode_tile = [&](const float* cX, int scatter_cnt, int64_t prefetch_tile, int prefetch_slot) {
#pragma unroll 1
    for (int jq = 0; jq < GPW / 2; ++jq) {
      if (scatter_cnt >= 0) scatter_group(md, a, GF, tmem_cache, jq, scatter_cnt, warp, lane);
      encode_group(cX, jq);
      if (jq == 0) {
        umma::fence_async_smem();
        __syncthreads();
        issue_z1(0, FE / 16, false);
      }
    }
    umma::tmem_st_wait();
    if (prefetch_tile < tiles)
      load_tile(a, prefetch_tile, sX + (prefetch_slot & 1) * 3 * P, sT + (prefetch_slot & 1) * P, tid);
    umma::fence_async_smem();
    umma::fence_before_sync();
    __syncthreads();  // F complete; every warp's scatter of the previous tile has read gF
    issue_z1(FE / 16, FE / 8, true);
  };

  int it = 0;
  if (int64_t(blockIdx.x) < tiles) encode_tile(sX, -1, int64_t(blockIdx.x) + gridDim.x, 1);
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++it) {
    const int cnt = int(min64(P, a.n - tile * P));
    const float* cT = sT + (it & 1) * P;
    TC_STAMP(0);
    TC_STAMP(1);
    umma::mbar_wait(bar, phase);
    phase ^= 1;
    umma::fence_after_sync();
    TC_STAMP(2);
    // ---- epilogue 1: h1 = relu(z1) -> h1 hi/lo; sign bitmap for the dz1 mask ----
    {
      float v[EPC];
      umma::tmem_ld16(TZ1 + lane_base + ep_col0, v);
      if (lane < 16) {
#pragma unroll
        for (int c4 = 0; c4 < EPC; c4 += 4) {
          float hi[4], lo[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) umma::split_tf32(fmaxf(v[c4 + e], 0.f), hi[e], lo[e]);
          const uint32_t o = cm64(ep_row, ep_col0 + c4);
          *reinterpret_cast<float4*>(H1h + o) = make_float4(hi[0], hi[1], hi[2], hi[3]);
          *reinterpret_cast<float4*>(H1l + o) = make_float4(lo[0], lo[1], lo[2], lo[3]);
        }
      }
#pragma unroll
      for (int c = 0; c < EPC; ++c) {
        const unsigned b = __ballot_sync(0xffffffffu, lane < 16 && v[c] > 0.f);
        if (lane == 0) sM1[(ep_col0 + c) * 4 + quarter] = uint16_t(b & 0xffffu);
      }
    }
    umma::fence_async_smem();
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    TC_STAMP(3);
    // ---- z2 = h1 W2^T (3xTF32) ----
    if (tid == 0) {
      for (int kk = 0; kk < HID / 8; ++kk) {
        const uint64_t hh = umma::desc_kmajor(sH1h, 64, kk), hl = umma::desc_kmajor(sH1l, 64, kk);
        const uint64_t wh = umma::desc_kmajor(sW2h, 64, kk), wl = umma::desc_kmajor(sW2l, 64, kk);
        umma::mma_tf32(TZ2, hh, wh, idesc64, kk > 0);
        umma::mma_tf32(TZ2, hh, wl, idesc64, 1);
        umma::mma_tf32(TZ2, hl, wh, idesc64, 1);
      }
      umma::commit(bar);
    }
    umma::mbar_wait(bar, phase);
    phase ^= 1;
    umma::fence_after_sync();
    TC_STAMP(4);
    // ---- epilogue 2: h2, head, loss, g, mask, dW3 ----
    float h2v[EPC];
    umma::tmem_ld16(TZ2 + lane_base + ep_col0, h2v);
    if (lane < 16) {
      float part = 0.f;
#pragma unroll
      for (int c = 0; c < EPC; ++c) {
        h2v[c] = fmaxf(h2v[c], 0.f);
        part = fmaf(h2v[c], sW3[ep_col0 + c], part);
      }
      sHead[wq * P + ep_row] = part;
#pragma unroll
      for (int c4 = 0; c4 < EPC; c4 += 4)
        *reinterpret_cast<float4*>(MASK + cm64(ep_row, ep_col0 + c4)) =
            make_float4(h2v[c4] > 0.f ? 1.f : 0.f, h2v[c4 + 1] > 0.f ? 1.f : 0.f, h2v[c4 + 2] > 0.f ? 1.f : 0.f,
                        h2v[c4 + 3] > 0.f ? 1.f : 0.f);
    }
    umma::fence_before_sync();
    __syncthreads();
    if (tid < P) {
      float g = 0.f;
      if (tid < cnt) {
        float raw = sHead[tid];
#pragma unroll
        for (int q = 1; q < WQ; ++q) raw += sHead[q * P + tid];
        const float y = __fadd_rn(__fmul_rn(raw, md.span), md.vmin);
        const float r = __fsub_rn(y, cT[tid]);
        const float s = __fmul_rn(r, r);
        a.sq[tile * P + tid] = s;
        loss += double(s);
        g = __fmul_rn(r, coef);
      }
      sG[tid] = g;
    }
    umma::fence_async_smem();
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    TC_STAMP(5);
    // ---- dz1^T[i][p] = sum_j V[i][j] mask[p][j]  (A = V from TMEM, 2 products) ----
    if (tid == 0) {
      for (int kk = 0; kk < HID / 8; ++kk) {
        const uint64_t mk = umma::desc_kmajor(sMask, 64, kk);
        umma::mma_tf32_ts(TZ1, tmem + TC_VH + 8 * kk, mk, idesc128, kk > 0);
        umma::mma_tf32_ts(TZ1, tmem + TC_VL + 8 * kk, mk, idesc128, 1);
      }
      umma::commit(bar);
    }
    if (lane < 16) {
      const float g = sG[ep_row];
#pragma unroll
      for (int c = 0; c < EPC; ++c) dw3_acc[c] = fmaf(g, h2v[c], dw3_acc[c]);
    }
    // dW2[j][i] += sum_p dz2[p][j] h1[p][i],  dz2[p][j] = mask[p][j] (g[p] w3[j])  (single TF32)
    if (!(a.skip & 2)) {
#pragma unroll 2
      for (int kk = 0; kk < 8; ++kk) {
        const int j0 = 16 * mt + gid, pk = 8 * kk + tig;
        const float g0 = sG[pk], g4 = sG[pk + 4], w0 = sW3[j0], w8 = sW3[j0 + 8];
        const uint32_t av[4] = {tf32_bits(MASK[cm64(pk, j0)] * __fmul_rn(g0, w0)),
                                tf32_bits(MASK[cm64(pk, j0 + 8)] * __fmul_rn(g0, w8)),
                                tf32_bits(MASK[cm64(pk + 4, j0)] * __fmul_rn(g4, w0)),
                                tf32_bits(MASK[cm64(pk + 4, j0 + 8)] * __fmul_rn(g4, w8))};
#pragma unroll
        for (int t = 0; t < NT64; ++t) {
          const int ic = 8 * (NT64 * wn + t) + gid;
          const uint32_t ob = kk * 32 + tig * 4 + cm_col(ic);
          const uint32_t bv[2] = {__float_as_uint(H1h[ob]), __float_as_uint(H1h[ob + 16])};
          mma_tf32_16x8x8(acc2[t], av, bv);
        }
      }
    }
    umma::mbar_wait(bar, phase);
    phase ^= 1;
    umma::fence_before_sync();
    __syncthreads();  // dW2 has consumed h1 before dz1 overwrites it
    umma::fence_after_sync();
    TC_STAMP(6);
    // ---- dz1 epilogue: row i = lane of quarter q (rows repeat every 64), 8 points per warp;
    // an 8x8 register transpose within lane octets turns the column-per-lane values into
    // row-per-lane float4 stores (CM rows are 16-byte chunks) ----
    {
      const int i = 32 * (quarter & 1) + lane, p0 = 8 * (wq + 4 * (quarter >> 1));
      float v[8];
      umma::tmem_ld8(TZ1 + lane_base + p0, v);
      const uint32_t bits = uint32_t(sM1[i * 4 + (p0 >> 4)]) >> (p0 & 15);
#pragma unroll
      for (int c = 0; c < 8; ++c) v[c] = ((bits >> c) & 1u) ? __fmul_rn(sG[p0 + c], v[c]) : 0.f;
      const int l = lane & 7;
#pragma unroll
      for (int st = 4; st >= 1; st >>= 1) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          if (c & st) continue;
          const bool up = l & st;
          const float r = __shfl_xor_sync(0xffffffffu, up ? v[c] : v[c ^ st], st);
          if (up)
            v[c] = r;
          else
            v[c ^ st] = r;
        }
      }
      // now v[c] = dz1[p0 + l][ib + c]
      const int p = p0 + l, ib = 32 * (quarter & 1) + (lane & ~7);
      float hi[8], lo[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) umma::split_tf32(v[c], hi[c], lo[c]);
      *reinterpret_cast<float4*>(DZ1h + cm64(p, ib)) = make_float4(hi[0], hi[1], hi[2], hi[3]);
      *reinterpret_cast<float4*>(DZ1h + cm64(p, ib + 4)) = make_float4(hi[4], hi[5], hi[6], hi[7]);
      *reinterpret_cast<float4*>(DZ1l + cm64(p, ib)) = make_float4(lo[0], lo[1], lo[2], lo[3]);
      *reinterpret_cast<float4*>(DZ1l + cm64(p, ib + 4)) = make_float4(lo[4], lo[5], lo[6], lo[7]);
    }
    umma::fence_async_smem();
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    TC_STAMP(7);
    // ---- gF^T[k][p] = sum_i W1^T[k][i] dz1[p][i]  (A = W1^T from TMEM, 3xTF32) ----
    if (tid == 0) {
      for (int kk = 0; kk < HID / 8; ++kk) {
        const uint64_t dh = umma::desc_kmajor(sH1h, 64, kk), dl = umma::desc_kmajor(sH1l, 64, kk);
        umma::mma_tf32_ts(TZ2, tmem + TC_W1TH + 8 * kk, dh, idesc128, kk > 0);
        umma::mma_tf32_ts(TZ2, tmem + TC_W1TH + 8 * kk, dl, idesc128, 1);
        umma::mma_tf32_ts(TZ2, tmem + TC_W1TL + 8 * kk, dh, idesc128, 1);
      }
      umma::commit(bar);
    }
    // dW1[i][k] += sum_p dz1[p][i] F[p][k]  (single TF32: the round-to-nearest hi parts)
    if (!(a.skip & 2)) {
#pragma unroll 2
      for (int kk = 0; kk < 8; ++kk) {
        const int i0 = 16 * mt + gid;
        const uint32_t oa = kk * 32 + tig * 4;
        const uint32_t av[4] = {__float_as_uint(DZ1h[oa + cm_col(i0)]), __float_as_uint(DZ1h[oa + cm_col(i0 + 8)]),
                                __float_as_uint(DZ1h[oa + 16 + cm_col(i0)]),
                                __float_as_uint(DZ1h[oa + 16 + cm_col(i0 + 8)])};
#pragma unroll
        for (int t = 0; t < NT128; ++t) {
          const int kc = 8 * (NT128 * wn + t) + gid;
          const uint32_t ob = oa + cm_col(kc);
          const uint32_t bv[2] = {__float_as_uint(Fh[ob]), __float_as_uint(Fh[ob + 16])};
          mma_tf32_16x8x8(acc1[t], av, bv);
        }
      }
    }
    umma::mbar_wait(bar, phase);
    phase ^= 1;
    umma::fence_before_sync();
    __syncthreads();  // dW1 and the gF^T product have consumed dz1 before gF overwrites it
    umma::fence_after_sync();
    TC_STAMP(8);
    // ---- gF epilogue: row k = lane of each quarter, 16 points per warp -> gF[p][k] ----
    {
      const int k = 32 * quarter + lane;
      float v[16];
      umma::tmem_ld16(TZ2 + lane_base + 16 * wq, v);
#pragma unroll
      for (int c = 0; c < 16; ++c) GF[gf_idx(16 * wq + c, k)] = v[c];
    }
    umma::fence_before_sync();
    __syncthreads();
    TC_STAMP(9);
    // ---- scatter of this tile, interleaved with the encode of the next one ----
    const int64_t next = tile + gridDim.x;
    if (next < tiles) {
      encode_tile(sX + ((it + 1) & 1) * 3 * P, cnt, next + gridDim.x, it + 2);
    } else {
#pragma unroll 1
      for (int jq = 0; jq < GPW / 2; ++jq) scatter_group(md, a, GF, tmem_cache, jq, cnt, warp, lane);
    }
    TC_STAMP(10);
  }

  // ---- flush per-CTA partials: [dW1 (64x128) | dW2 (64x64) | dW3 (64)] ----
  float* dst = a.part_dw + int64_t(blockIdx.x) * (HID * FE + HID * HID + HID);
  {
#pragma unroll
    for (int t = 0; t < NT128; ++t) {
      const int c0 = 8 * (NT128 * wn + t) + 2 * tig, r0 = 16 * mt + gid;
      dst[r0 * FE + c0] = acc1[t][0];
      dst[r0 * FE + c0 + 1] = acc1[t][1];
      dst[(r0 + 8) * FE + c0] = acc1[t][2];
      dst[(r0 + 8) * FE + c0 + 1] = acc1[t][3];
    }
    float* d2 = dst + HID * FE;
#pragma unroll
    for (int t = 0; t < NT64; ++t) {
      const int c0 = 8 * (NT64 * wn + t) + 2 * tig, r0 = 16 * mt + gid;
      d2[r0 * HID + c0] = acc2[t][0];
      d2[r0 * HID + c0 + 1] = acc2[t][1];
      d2[(r0 + 8) * HID + c0] = acc2[t][2];
      d2[(r0 + 8) * HID + c0 + 1] = acc2[t][3];
    }
  }
  if (lane < 16) {
#pragma unroll
    for (int c = 0; c < EPC; ++c) atomicAdd(&sDW3[ep_col0 + c], dw3_acc[c]);
  }
  const double bl = block_sum(loss, red);  // contains __syncthreads
  if (tid < HID) dst[HID * FE + HID * HID + tid] = sDW3[tid];
  if (tid == 0) a.part_loss[blockIdx.x] = bl;
  umma::fence_before_sync();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tmem, TMEM_COLS);
}

}  // namespace tc

extern "C" int apmg_debug_tc_phases(long long* out) {
  APMG_CUDA_TRY(cudaMemcpyFromSymbol(out, tc::g_tc_stamp, sizeof(tc::g_tc_stamp)));
  return APMG_OK;
}

bool recon_tc_eligible(const ModelDev<float>& md) {
  const char* e = getenv("APMG_MLP");  // APMG_MLP=simt forces the SIMT kernel (A/B tests)
  const bool tc_on = !(e && e[0] == 's');
  return tc_on && md.F == 128 && md.C == 2 && md.M == 64;
}

int launch_recon_tc(const ModelDev<float>& md, int64_t n, const float* coords, const float* targets, float* sq,
                    float* dgrid, float* part_dw, double* part_loss, int grid, const TrainCtl* ctl,
                    cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    APMG_CUDA_TRY(cudaFuncSetAttribute(tc::k_recon_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(tc::SMEM_BYTES)));
    attr = true;
  }
  const char* ea = getenv("APMG_SCATTER_AGG");
  const char* es = getenv("APMG_TC_SKIP");
  tc::Args a{md, n, coords, targets, sq, dgrid, part_dw, part_loss, ctl, (ea && ea[0] == '0') ? 0 : 1,
             es ? atoi(es) : 0};
  APMG_LAUNCH("recon_fwd_bwd_tc", tc::k_recon_tc, grid, tc::NT, tc::SMEM_BYTES, st, a);
  return APMG_OK;
}

}  // namespace apmg
