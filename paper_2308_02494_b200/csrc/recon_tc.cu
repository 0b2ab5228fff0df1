// Fused reconstruction step (optim.py:102-155) for the flagship shape
// (float32, 64 grids x 2 channels -> 128 features, 64 hidden), tensor-core MLP.
//
// One persistent CTA per SM; a 64-point tile per loop iteration:
//   encode      (point, grid) pairs -> features F, split hi/lo (3xTF32) in smem
//   z1 = F W1^T  tcgen05.mma kind::tf32, M=64 N=64 K=128, 3 products, TMEM accumulator
//   h1 = relu    tcgen05.ld epilogue -> h1 hi/lo in smem
//   z2 = h1 W2^T tcgen05.mma, M=64 N=64 K=64, 3 products
//   head/loss    epilogue: out = h2 w3 * span + vmin, residual, sq error, dL/dout, dz2
//   backward     register-fragment tensor MMAs (mma.sync m16n8k8 tf32):
//                 dz1 = (dz2 W2) * [z1>0]        3xTF32
//                 dW2 += dz2^T h1, dW1 += dz1^T F single TF32 (round-to-nearest operands)
//                 gF = dz1 W1                     3xTF32
//   scatter     d features -> channel-last grid gradients (float2 RED)
// Operands of the tcgen05 products are staged in the "CM" core-matrix layout of
// umma.cuh and consumed K-major; the backward needs transposed operands, which the
// register-fragment MMAs read directly from the same buffers.
#include "kernels.cuh"
#include "umma.cuh"

namespace apmg {
namespace tc {

constexpr int P = 64;        // points per tile (M of the tcgen05 products)
#ifndef APMG_TC_WARPS
#define APMG_TC_WARPS 16
#endif
constexpr int NW = APMG_TC_WARPS;  // warps per CTA (8 or 16)
constexpr int NT = 32 * NW;
constexpr int WQ = NW / 4;         // warps sharing one TMEM lane quarter
constexpr int EPC = 64 / WQ;       // accumulator columns per warp in the epilogues
constexpr int GPW = 64 / NW;       // grids per warp in encode / scatter
constexpr int MT_N64 = 32 / NW;    // 16x8 n-tiles per warp, 64-wide products
constexpr int MT_N128 = 64 / NW;   // 16x8 n-tiles per warp, 128-wide products
static_assert(NW == 8 || NW == 16, "tile mappings assume 8 or 16 warps");
constexpr int FE = 128;      // features
constexpr int HID = 64;
constexpr int DZS = 68;      // row stride (floats) of the plain dz2 buffer
constexpr int GFS = 132;     // row stride of the gF scatter buffer

// shared memory map (bytes)
constexpr uint32_t OFF_W1H = 0;
constexpr uint32_t OFF_W1L = OFF_W1H + 64 * 128 * 4;
constexpr uint32_t OFF_W2H = OFF_W1L + 64 * 128 * 4;
constexpr uint32_t OFF_W2L = OFF_W2H + 64 * 64 * 4;
constexpr uint32_t OFF_FH = OFF_W2L + 64 * 64 * 4;
constexpr uint32_t OFF_FL = OFF_FH + P * FE * 4;
constexpr uint32_t OFF_H1H = OFF_FL + P * FE * 4;
constexpr uint32_t OFF_H1L = OFF_H1H + P * HID * 4;  // later: dz1 (swizzled, stride 64)
// gF scatter buffer [P][GFS] reuses the h1 hi/lo region (h1 and dz1 are dead once gF is formed)
constexpr uint32_t GF_BYTES = (P * GFS * 4 > 2 * P * HID * 4) ? P * GFS * 4 : 2 * P * HID * 4;
constexpr uint32_t OFF_DZ2 = OFF_H1H + GF_BYTES;
constexpr uint32_t OFF_X = OFF_DZ2 + P * DZS * 4;
constexpr uint32_t OFF_T = OFF_X + P * 3 * 4;
constexpr uint32_t OFF_G = OFF_T + P * 4;
constexpr uint32_t OFF_HEAD = OFF_G + P * 4;         // [WQ][P] head partial sums
constexpr uint32_t OFF_DW3 = OFF_HEAD + WQ * P * 4;  // [64]
constexpr uint32_t OFF_RED = OFF_DW3 + HID * 4;      // [32] doubles
constexpr uint32_t OFF_BAR = OFF_RED + 32 * 8;
constexpr uint32_t OFF_TM = OFF_BAR + 8;
constexpr uint32_t OFF_TF = OFF_TM + 16;             // [64][12] transforms (f32)
constexpr uint32_t OFF_W3 = OFF_TF + 64 * 12 * 4;    // [64]
constexpr uint32_t SMEM_BYTES = OFF_W3 + 64 * 4;
constexpr uint32_t TMEM_COLS = 512;                  // z1 | z2 | cell cache, double-buffered (2 x 128)

__device__ __forceinline__ float* fptr(unsigned char* sm, uint32_t off) { return reinterpret_cast<float*>(sm + off); }

// float index of column c in a 64-row CM buffer (row part: (r/8)*32 + (r%8)*4)
__device__ __forceinline__ uint32_t cm_col(int c) { return uint32_t((c >> 2) * 256 + (c & 3)); }

// dz1 storage (stride 64, XOR swizzle on 4-float groups to keep fragment loads conflict-free)
__device__ __forceinline__ int dz1_idx(int p, int i) { return p * 64 + (i ^ ((p & 7) << 2)); }

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

// split an f32 fragment into (hi, lo) tf32 fragments
__device__ __forceinline__ void split_frag(const float* v, int n, uint32_t* hi, uint32_t* lo) {
  for (int e = 0; e < n; ++e) {
    hi[e] = tf32_bits(v[e]);
    lo[e] = tf32_bits(v[e] - __uint_as_float(hi[e]));
  }
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
  int skip;       // timing breakdown only (APMG_TC_SKIP): 1 scatter, 2 backward MMAs, 4 gathers
};

// Grid-gradient scatter of one tile: thread (warp, lane) owns points lane, lane + 32 and
// grids warp + NW*j, exactly the items it encoded; their cell terms come back from its TMEM
// cache, their feature gradients from GF [P][GFS].
__device__ __forceinline__ void scatter_tile(const ModelDev<float>& md, const Args& a, const float* GF,
                                             uint32_t tmem_cache, int cnt, int warp, int lane) {
#pragma unroll 1
  for (int jq = 0; jq < (a.skip & 1 ? 0 : GPW / 2); ++jq) {
    uint32_t cache[16];
    umma::tmem_ld16u(tmem_cache + 16 * jq, cache);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = 2 * jq + (u >> 1), h = u & 1;
      const int m = warp + NW * j, p = lane + 32 * h;
      const int vbase = int(cache[4 * u]);
      const bool valid = vbase >= 0 && p < cnt;
      float2 g = make_float2(0.f, 0.f);
      if (valid) g = *reinterpret_cast<const float2*>(GF + p * GFS + 2 * m);
      if (a.aggregate)
        scatter_vertex_warp_agg(md, a.dgrid, valid, vbase, __uint_as_float(cache[4 * u + 1]),
                                __uint_as_float(cache[4 * u + 2]), __uint_as_float(cache[4 * u + 3]), g.x, g.y);
      else if (valid)
        scatter_vertex_f32(md, a.dgrid, vbase, __uint_as_float(cache[4 * u + 1]), __uint_as_float(cache[4 * u + 2]),
                           __uint_as_float(cache[4 * u + 3]), g.x, g.y);
    }
  }
}

__global__ void __launch_bounds__(NT, 1) k_recon_tc(Args a) {
  extern __shared__ __align__(1024) unsigned char sm[];
  if (a.ctl && a.ctl->skip) return;
  const ModelDev<float>& md = a.md;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  float* W1h = fptr(sm, OFF_W1H);
  float* W1l = fptr(sm, OFF_W1L);
  float* W2h = fptr(sm, OFF_W2H);
  float* W2l = fptr(sm, OFF_W2L);
  float* Fh = fptr(sm, OFF_FH);
  float* Fl = fptr(sm, OFF_FL);
  float* H1h = fptr(sm, OFF_H1H);
  float* H1l = fptr(sm, OFF_H1L);
  float* DZ1 = fptr(sm, OFF_H1L);  // reuses h1_lo after the z2 product
  float* DZ2 = fptr(sm, OFF_DZ2);
  float* GF = fptr(sm, OFF_H1H);   // reuses h1/dz1 after gF (read by the next tile's scatter)
  float* sX = fptr(sm, OFF_X);
  float* sT = fptr(sm, OFF_T);
  float* sG = fptr(sm, OFF_G);
  float* sHead = fptr(sm, OFF_HEAD);
  float* sDW3 = fptr(sm, OFF_DW3);
  double* red = reinterpret_cast<double*>(sm + OFF_RED);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + OFF_BAR);
  uint32_t* tm_slot = reinterpret_cast<uint32_t*>(sm + OFF_TM);

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
  float* sTF = fptr(sm, OFF_TF);
  for (int e = tid; e < 64 * 12; e += NT) sTF[e] = md.tf[16 * (e / 12) + (e % 12)];
  float* sW3 = fptr(sm, OFF_W3);
  if (tid < HID) sW3[tid] = md.w3[tid];
  if (warp == 0) umma::tmem_alloc(tm_slot, TMEM_COLS);
  if (tid == 0) {
    umma::mbar_init(bar, 1);
    umma::fence_mbar_init();
  }
  umma::fence_async_smem();
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tmem = *tm_slot;
  const uint32_t TZ1 = tmem, TZ2 = tmem + 64;
  // this warp's lane quarter; the WQ warps sharing it use disjoint 8*GPW-column slices;
  // buffer (tile parity) b at +128*b: encode(t) fills one while scatter(t-1) drains the other
  const uint32_t tmem_cache0 = tmem + 128 + 8 * GPW * (warp >> 2) + (uint32_t(32 * (warp & 3)) << 16);
  const uint32_t sW1h = umma::smem_u32(W1h), sW1l = umma::smem_u32(W1l), sW2h = umma::smem_u32(W2h),
                 sW2l = umma::smem_u32(W2l), sFh = umma::smem_u32(Fh), sFl = umma::smem_u32(Fl),
                 sH1h = umma::smem_u32(H1h), sH1l = umma::smem_u32(H1l);
  const uint32_t idesc64 = umma::idesc_tf32(64, 64, false, false);
  const float coef = __fmul_rn(float(2.0 / double(a.n)), md.span);

  // persistent weight-gradient accumulators (mma.sync fragments); warp w owns m-tile
  // mt = w / WQ (16 rows) and a contiguous run of 8-column n-tiles
  const int mt = warp / WQ, wn = warp % WQ;
  float acc1[MT_N128][4];  // dW1 [64 i][128 k]: n-tiles MT_N128*wn ..
  float acc2[MT_N64][4];   // dW2 [64 j][64 i]:  n-tiles MT_N64*wn ..
#pragma unroll
  for (int t = 0; t < MT_N128; ++t)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc1[t][e] = 0.f;
#pragma unroll
  for (int t = 0; t < MT_N64; ++t)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc2[t][e] = 0.f;
  float dw3_acc[EPC];
#pragma unroll
  for (int c = 0; c < EPC; ++c) dw3_acc[c] = 0.f;
  double loss = 0.0;
  uint32_t phase = 0;

  // TMEM epilogue mapping (M=64 accumulator: row 16*(w%4)+t lives in lane 32*(w%4)+t, t < 16)
  const int ep_row = 16 * (warp & 3) + lane;  // valid when lane < 16
  const int ep_col0 = EPC * (warp >> 2);       // the WQ warps of a quarter split the 64 columns
  const uint32_t ep_lane = uint32_t(32 * (warp & 3)) << 16;

  const int64_t tiles = ceil_div(a.n, P);
  // Software pipeline: the scatter of tile t-1 (atomics, shuffles) runs while the tensor
  // core forms z1 of tile t; its gF rows live in the h1 region until epilogue 1 of tile t.
  int prev_cnt = 0;
  for (int64_t tile = blockIdx.x, it = 0;; tile += gridDim.x, ++it) {
    const bool have = tile < tiles;
    if (!have) {
      if (it > 0) scatter_tile(md, a, GF, tmem_cache0 + 128 * uint32_t((it - 1) & 1), prev_cnt, warp, lane);
      break;
    }
    const uint32_t tmem_cache = tmem_cache0 + 128 * uint32_t(it & 1);
    const int64_t p0 = tile * P;
    const int cnt = int(min64(P, a.n - p0));
    if (tid < P) {
      const bool ok = tid < cnt;
      const int64_t i = p0 + tid;
      sX[3 * tid] = ok ? a.coords[3 * i] : 0.f;
      sX[3 * tid + 1] = ok ? a.coords[3 * i + 1] : 0.f;
      sX[3 * tid + 2] = ok ? a.coords[3 * i + 2] : 0.f;
      sT[tid] = ok ? a.targets[i] : 0.f;
    }
    __syncthreads();
    // ---- encode: lane -> point, warp -> grid; cell terms cached in TMEM for the scatter ----
    {
      const float xa[2][3] = {{sX[3 * lane], sX[3 * lane + 1], sX[3 * lane + 2]},
                              {sX[3 * (lane + 32)], sX[3 * (lane + 32) + 1], sX[3 * (lane + 32) + 2]}};
#pragma unroll 1
      for (int jq = 0; jq < GPW / 2; ++jq) {  // groups of (2 grids x 2 points)
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
      }
      umma::tmem_st_wait();
    }
    umma::fence_async_smem();
    __syncthreads();
    // ---- z1 = F W1^T (3xTF32) ----
    if (tid == 0) {
      umma::fence_after_sync();
      for (int kk = 0; kk < FE / 8; ++kk) {
        const uint64_t fh = umma::desc_kmajor(sFh, 64, kk), fl = umma::desc_kmajor(sFl, 64, kk);
        const uint64_t wh = umma::desc_kmajor(sW1h, 64, kk), wl = umma::desc_kmajor(sW1l, 64, kk);
        umma::mma_tf32(TZ1, fh, wh, idesc64, kk > 0);
        umma::mma_tf32(TZ1, fh, wl, idesc64, 1);
        umma::mma_tf32(TZ1, fl, wh, idesc64, 1);
      }
      umma::commit(bar);
    }
    if (it > 0) scatter_tile(md, a, GF, tmem_cache0 + 128 * uint32_t((it - 1) & 1), prev_cnt, warp, lane);
    umma::mbar_wait(bar, phase);
    phase ^= 1;
    umma::fence_before_sync();
    __syncthreads();  // every warp's scatter has consumed GF before epilogue 1 overwrites it
    umma::fence_after_sync();
    // ---- epilogue 1: h1 = relu(z1) -> H1 hi/lo ----
    {
      float v[EPC];
#pragma unroll
      for (int c = 0; c < EPC; c += 16) umma::tmem_ld16(TZ1 + ep_lane + ep_col0 + c, v + c);
      if (lane < 16) {
#pragma unroll
        for (int c4 = 0; c4 < EPC; c4 += 4) {
          float hi[4], lo[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) umma::split_tf32(fmaxf(v[c4 + e], 0.f), hi[e], lo[e]);
          const uint32_t o = umma::cm_offset(ep_row, ep_col0 + c4, 64) >> 2;
          *reinterpret_cast<float4*>(H1h + o) = make_float4(hi[0], hi[1], hi[2], hi[3]);
          *reinterpret_cast<float4*>(H1l + o) = make_float4(lo[0], lo[1], lo[2], lo[3]);
        }
      }
    }
    umma::fence_async_smem();
    umma::fence_before_sync();
    __syncthreads();
    // ---- z2 = h1 W2^T (3xTF32) ----
    if (tid == 0) {
      umma::fence_after_sync();
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
    // ---- epilogue 2: h2, head, loss, dz2, dW3 ----
    float h2v[EPC];
#pragma unroll
    for (int c = 0; c < EPC; c += 16) umma::tmem_ld16(TZ2 + ep_lane + ep_col0 + c, h2v + c);
    if (lane < 16) {
      float part = 0.f;
#pragma unroll
      for (int c = 0; c < EPC; ++c) {
        h2v[c] = fmaxf(h2v[c], 0.f);
        part = fmaf(h2v[c], sW3[ep_col0 + c], part);
      }
      sHead[(warp >> 2) * P + ep_row] = part;
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
        const float r = __fsub_rn(y, sT[tid]);
        const float s = __fmul_rn(r, r);
        a.sq[p0 + tid] = s;
        loss += double(s);
        g = __fmul_rn(r, coef);
      }
      sG[tid] = g;
    }
    __syncthreads();
    if (lane < 16) {
      const float g = sG[ep_row];
#pragma unroll
      for (int c = 0; c < EPC; ++c) {
        const float hv = h2v[c];
        dw3_acc[c] = fmaf(g, hv, dw3_acc[c]);
        DZ2[ep_row * DZS + ep_col0 + c] = hv > 0.f ? __fmul_rn(g, sW3[ep_col0 + c]) : 0.f;
      }
    }
    __syncthreads();
    // ---- backward 1: dz1 = (dz2 W2) * [h1 > 0]  (M=64 p, N=64 i, K=64 j), 3xTF32 ----
    if (!(a.skip & 2)) {
      const int nt0 = MT_N64 * wn;
      float d[MT_N64][4];
#pragma unroll
      for (int t = 0; t < MT_N64; ++t)
#pragma unroll
        for (int e = 0; e < 4; ++e) d[t][e] = 0.f;
#pragma unroll 2
      for (int kk = 0; kk < 8; ++kk) {
        const int r0 = 16 * mt + gid, k0 = 8 * kk + tig;
        float av[4] = {DZ2[r0 * DZS + k0], DZ2[(r0 + 8) * DZS + k0], DZ2[r0 * DZS + k0 + 4],
                       DZ2[(r0 + 8) * DZS + k0 + 4]};
        uint32_t ah[4], al[4];
        split_frag(av, 4, ah, al);
#pragma unroll
        for (int t = 0; t < MT_N64; ++t) {
          const int ncol = 8 * (nt0 + t) + gid;  // i
          const uint32_t o0 = kk * 32 + tig * 4 + cm_col(ncol), o1 = o0 + 16;
          const uint32_t bh[2] = {__float_as_uint(W2h[o0]), __float_as_uint(W2h[o1])};
          const uint32_t bl[2] = {__float_as_uint(W2l[o0]), __float_as_uint(W2l[o1])};
          mma_tf32_16x8x8(d[t], ah, bh);
          mma_tf32_16x8x8(d[t], ah, bl);
          mma_tf32_16x8x8(d[t], al, bh);
        }
      }
#pragma unroll
      for (int t = 0; t < MT_N64; ++t) {
        const int c0 = 8 * (nt0 + t) + 2 * tig;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int pr = 16 * mt + gid + ((e & 2) ? 8 : 0), ic = c0 + (e & 1);
          const float hv = H1h[umma::cm_offset(pr, ic, 64) >> 2];
          DZ1[dz1_idx(pr, ic)] = hv > 0.f ? d[t][e] : 0.f;
        }
      }
    }
    __syncthreads();
    // ---- backward 2: weight gradients (single TF32, round-to-nearest operands) ----
    if (!(a.skip & 2)) {
      // dW2[j][i] += sum_p dz2[p][j] h1[p][i]   (A = dz2^T, B = h1)
#pragma unroll 2
      for (int kk = 0; kk < 8; ++kk) {
        const int j0 = 16 * mt + gid, pk = 8 * kk + tig;
        const uint32_t av[4] = {tf32_bits(DZ2[pk * DZS + j0]), tf32_bits(DZ2[pk * DZS + j0 + 8]),
                                tf32_bits(DZ2[(pk + 4) * DZS + j0]), tf32_bits(DZ2[(pk + 4) * DZS + j0 + 8])};
#pragma unroll
        for (int t = 0; t < MT_N64; ++t) {
          const int ic = 8 * (MT_N64 * wn + t) + gid;
          const uint32_t ob = kk * 32 + tig * 4 + cm_col(ic);
          const uint32_t bv[2] = {__float_as_uint(H1h[ob]), __float_as_uint(H1h[ob + 16])};
          mma_tf32_16x8x8(acc2[t], av, bv);
        }
      }
      // dW1[i][k] += sum_p dz1[p][i] F[p][k]    (A = dz1^T, B = F)
#pragma unroll 2
      for (int kk = 0; kk < 8; ++kk) {
        const int i0 = 16 * mt + gid, pk = 8 * kk + tig;
        const uint32_t av[4] = {tf32_bits(DZ1[dz1_idx(pk, i0)]), tf32_bits(DZ1[dz1_idx(pk, i0 + 8)]),
                                tf32_bits(DZ1[dz1_idx(pk + 4, i0)]), tf32_bits(DZ1[dz1_idx(pk + 4, i0 + 8)])};
#pragma unroll
        for (int t = 0; t < MT_N128; ++t) {
          const int kc = 8 * (MT_N128 * wn + t) + gid;
          const uint32_t ob = kk * 32 + tig * 4 + cm_col(kc);
          const uint32_t bv[2] = {__float_as_uint(Fh[ob]), __float_as_uint(Fh[ob + 16])};
          mma_tf32_16x8x8(acc1[t], av, bv);
        }
      }
    }
    __syncthreads();
    // ---- backward 3: gF = dz1 W1 (M=64 p, N=128 k, K=64 i), 3xTF32, into the F region ----
    if (!(a.skip & 2)) {
      const int nt0 = MT_N128 * wn;
      float d[MT_N128][4];
#pragma unroll
      for (int t = 0; t < MT_N128; ++t)
#pragma unroll
        for (int e = 0; e < 4; ++e) d[t][e] = 0.f;
#pragma unroll 1
      for (int kk = 0; kk < 8; ++kk) {
        const int r0 = 16 * mt + gid, k0 = 8 * kk + tig;
        float av[4] = {DZ1[dz1_idx(r0, k0)], DZ1[dz1_idx(r0 + 8, k0)], DZ1[dz1_idx(r0, k0 + 4)],
                       DZ1[dz1_idx(r0 + 8, k0 + 4)]};
        uint32_t ah[4], al[4];
        split_frag(av, 4, ah, al);
#pragma unroll
        for (int t = 0; t < MT_N128; ++t) {
          const int kc = 8 * (nt0 + t) + gid;  // feature column
          const uint32_t o0 = kk * 32 + tig * 4 + cm_col(kc), o1 = o0 + 16;
          const uint32_t bh[2] = {__float_as_uint(W1h[o0]), __float_as_uint(W1h[o1])};
          const uint32_t bl[2] = {__float_as_uint(W1l[o0]), __float_as_uint(W1l[o1])};
          mma_tf32_16x8x8(d[t], ah, bh);
          mma_tf32_16x8x8(d[t], ah, bl);
          mma_tf32_16x8x8(d[t], al, bh);
        }
      }
      __syncthreads();  // all warps done reading dz1 / h1 before gF overwrites them
#pragma unroll
      for (int t = 0; t < MT_N128; ++t) {
        const int c0 = 8 * (nt0 + t) + 2 * tig, pr = 16 * mt + gid;
        *reinterpret_cast<float2*>(GF + pr * GFS + c0) = make_float2(d[t][0], d[t][1]);
        *reinterpret_cast<float2*>(GF + (pr + 8) * GFS + c0) = make_float2(d[t][2], d[t][3]);
      }
    }
    __syncthreads();
    prev_cnt = cnt;
  }

  // ---- flush per-CTA partials: [dW1 (64x128) | dW2 (64x64) | dW3 (64)] ----
  float* dst = a.part_dw + int64_t(blockIdx.x) * (HID * FE + HID * HID + HID);
  {
#pragma unroll
    for (int t = 0; t < MT_N128; ++t) {
      const int c0 = 8 * (MT_N128 * wn + t) + 2 * tig, r0 = 16 * mt + gid;
      dst[r0 * FE + c0] = acc1[t][0];
      dst[r0 * FE + c0 + 1] = acc1[t][1];
      dst[(r0 + 8) * FE + c0] = acc1[t][2];
      dst[(r0 + 8) * FE + c0 + 1] = acc1[t][3];
    }
    float* d2 = dst + HID * FE;
#pragma unroll
    for (int t = 0; t < MT_N64; ++t) {
      const int c0 = 8 * (MT_N64 * wn + t) + 2 * tig, r0 = 16 * mt + gid;
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
