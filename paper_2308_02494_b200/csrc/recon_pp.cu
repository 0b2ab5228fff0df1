// Fused reconstruction step (optim.py:102-155), flagship shape (float32, 64 grids x 2 channels ->
// 128 features, 64 hidden), as two ping-ponged worker groups per SM.
//
// The chain of one tile -- encode -> z1 -> h1 -> z2 -> head/loss -> dz2 -> dz1 || dW2 -> dz1 mask ->
// gF || dW1 -> gF -> scatter -- is serial, and at a single group per SM the tensor-core steps and
// the epilogues expose the CUDA cores' idle time and the warps' barrier waits.  Here one CTA per
// SM holds two independent groups of 8 warps, each running that chain on its own 32-point tiles
// with its own operand buffers and TMEM accumulators: while one group waits on the tensor core or
// a barrier, the other group's encode / scatter keeps the SM busy.  Nothing is interleaved by
// hand; each group's code is straight-line.  A group's products are issued by one thread of its
// warp 7, which has no accumulator rows to read in the epilogues (16 warps in all: 4 per SM
// sub-partition, so the register budget stays at 128 per thread).
//
// Tiles are 32 points (lane = point: a warp encodes / scatters 8 grids of all 32 points of its
// group's tile, the 16 features of a point are 2 conflict-free 16-byte stores per plane).  The
// products are M=64: rows 0-31 are the tile, rows 32-63 read the buffer's next K chunk (results
// discarded); the buffers use the 32-row core-matrix layout, so a group needs half the shared
// memory of a 64-point tile and both groups fit with the bf16x3 operands of the tc16 kernel:
//   z1 = F W1^T   6 products (bf16x3: f32-level forward)   z2 = h1 W2^T   6 products
//   dz1 = dz2 W2, dW2 += dz2^T h1, gF = dz1 W1, dW1 += dz1^T F   3 products each (~2^-16)
// The cell terms of the scatter are recomputed from the point (kept in registers) instead of
// being cached: exact f32 fractions, and TMEM holds only accumulators:
//   per group: acc A (z1, dz1) | acc B (z2) (gF spans both)  x 2  +  dW1 | dW2 (shared)  = 448 cols
#include "kernels.cuh"
#include "umma.cuh"

namespace apmg {
namespace pp {

constexpr int P = 32;             // points per group tile
constexpr int NG = 2;             // worker groups
constexpr int GW = 8;             // warps per group
constexpr int GT = 32 * GW;       // threads per group
constexpr int NWK = NG * GW;      // worker warps
constexpr int NTA = 32 * NWK;
constexpr int ISSUER = 7;         // the warp of a group whose lane 0 issues the group's products
constexpr int FE = 128, HID = 64;

constexpr uint32_t PLW1 = 64 * FE * 2, PLW2 = 64 * HID * 2;  // weight planes (64 rows)
constexpr uint32_t PLF = P * FE * 2, PLH = P * HID * 2;       // 32-row operand planes
// rows 32..63 of an M=64 product read 512 B (4 core-matrix groups) past the buffer's K chunk
constexpr uint32_t SLACK = 512;
constexpr uint32_t OFF_W1 = 0;
constexpr uint32_t OFF_W2 = OFF_W1 + 3 * PLW1;
constexpr uint32_t OFF_GRP = OFF_W2 + 3 * PLW2;
// per group: F (3 planes; the f32 gF [32][128] overlays it once dW1 has consumed F) | h1 (3) |
// dz (2 planes: dz2, then dz1 once dz1 || dW2 have consumed dz2) | slack
constexpr uint32_t G_F = 0, G_H1 = G_F + 3 * PLF, G_DZ = G_H1 + 3 * PLH, G_BYTES = G_DZ + 2 * PLH + SLACK;
static_assert(P * FE * 4 <= 3 * PLF, "gF overlays F");
constexpr uint32_t OFF_TF = OFF_GRP + NG * G_BYTES;       // [64][12] transforms (f32)
constexpr uint32_t OFF_DET = OFF_TF + 64 * 12 * 4;        // [64] |det A| (fused density)
constexpr uint32_t OFF_W3 = OFF_DET + 64 * 4;             // [64]
constexpr uint32_t OFF_RHO = OFF_W3 + 64 * 4;             // [NG][GW][P] per-warp partial rho
constexpr uint32_t OFF_HEAD = OFF_RHO + NG * GW * P * 4;  // [NG][2][P] partial heads per column half
constexpr uint32_t OFF_DW3 = OFF_HEAD + NG * 2 * P * 4;   // [NG * 2 quarters][64]
constexpr uint32_t OFF_RED = OFF_DW3 + NG * 2 * HID * 4;  // [32] doubles
constexpr uint32_t OFF_BAR = OFF_RED + 32 * 8;            // [NG][8] mbarriers
constexpr uint32_t OFF_TM = OFF_BAR + NG * 8 * 8;
constexpr uint32_t SMEM_BYTES = OFF_TM + 16;
static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");

constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t TC_DW1 = 256, TC_DW2 = 384;  // group g: acc A at 128 g, acc B at 128 g + 64

// mbarriers of a group: operands ready (epilogue warps -> issuer) and products done (commit -> workers)
enum { B_H1 = 0, B_DZ2, B_DZ1, B_Z1, B_Z2, B_D1, B_GF };

// bf16x3 product q: (A plane, B plane) = hh, hm, mh, hl, lh, mm
__host__ __device__ constexpr int kPA(int q) { return q == 2 ? 1 : (q == 4 ? 2 : (q == 5 ? 1 : 0)); }
__host__ __device__ constexpr int kPB(int q) { return q == 1 ? 1 : (q == 3 ? 2 : (q == 5 ? 1 : 0)); }

__device__ __forceinline__ float ex2_ftz(float v) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}

// flat-top bump exp(-sum_d l_d^20) (density.py:83-103, p = 10) of two (point, grid) pairs in packed
// fp32x2, the arithmetic of k_dens_rho32x2 (l^2 clamped at 4)
__device__ __forceinline__ float2 bump_p10x2(float2 l0, float2 l1, float2 l2) {
  const float2 la[3] = {l0, l1, l2};
  float2 acc = make_float2(0.f, 0.f);
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    float2 s = __fmul2_rn(la[d], la[d]);
    s = make_float2(fminf(s.x, 4.f), fminf(s.y, 4.f));
    const float2 s2 = __fmul2_rn(s, s), s4 = __fmul2_rn(s2, s2), s8 = __fmul2_rn(s4, s4);
    acc = __ffma2_rn(__fmul2_rn(s8, s), s, acc);
  }
  const float2 e = __fmul2_rn(acc, make_float2(-1.4426950408889634f, -1.4426950408889634f));
  return make_float2(ex2_ftz(e.x), ex2_ftz(e.y));
}

// local coordinate axis of one point in two grids: ((x0 a0 + x1 a1) + x2 a2) + t per grid, each
// product rounded on its own (model.py:179-182 in f32; the products stay scalar so no add is
// contracted into them), the sums packed
__device__ __forceinline__ float2 local_axis_g2(float x0, float x1, float x2, const float* ta, const float* tb) {
  const float2 p0 = make_float2(__fmul_rn(x0, ta[0]), __fmul_rn(x0, tb[0]));
  const float2 p1 = make_float2(__fmul_rn(x1, ta[1]), __fmul_rn(x1, tb[1]));
  const float2 p2 = make_float2(__fmul_rn(x2, ta[2]), __fmul_rn(x2, tb[2]));
  return __fadd2_rn(__fadd2_rn(__fadd2_rn(p0, p1), p2), make_float2(ta[3], tb[3]));
}

// gF [32][128] f32, 16-byte chunks XOR-swizzled by row (chunk ^ (row & 7)): the scatter's row-per-lane
// 16-byte reads and the epilogue's 8-byte writes both spread over the banks
__device__ __forceinline__ int gf_idx(int row, int col) {
  return row * FE + ((((col >> 2) ^ (row & 7)) << 2) | (col & 3));
}

__device__ __forceinline__ bool mbar_test(uint64_t* mbar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(ok)
      : "r"(umma::smem_u32(mbar)), "r"(parity)
      : "memory");
  return ok != 0;
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
};

// tiles of group g of CTA b: 2 b + g + i * 2 gridDim
__device__ __forceinline__ int64_t group_tiles(int64_t tiles, int g) {
  const int64_t first = 2 * int64_t(blockIdx.x) + g, stride = 2 * int64_t(gridDim.x);
  return first < tiles ? (tiles - first + stride - 1) / stride : 0;
}

template <bool FX>  // FX: deterministic training (fixed-point grid gradient)
__global__ void __launch_bounds__(NTA, 1) k_recon_pp(Args a) {
  extern __shared__ __align__(1024) unsigned char sm[];
  if (a.ctl && a.ctl->skip) return;
  const ModelDev<float>& md = a.md;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float* sTF = reinterpret_cast<float*>(sm + OFF_TF);
  float* sDET = reinterpret_cast<float*>(sm + OFF_DET);
  float* sW3 = reinterpret_cast<float*>(sm + OFF_W3);
  float* sRHO = reinterpret_cast<float*>(sm + OFF_RHO);
  float* sHead = reinterpret_cast<float*>(sm + OFF_HEAD);
  float* sDW3 = reinterpret_cast<float*>(sm + OFF_DW3);
  double* red = reinterpret_cast<double*>(sm + OFF_RED);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + OFF_BAR);
  uint32_t* tm_slot = reinterpret_cast<uint32_t*>(sm + OFF_TM);
  const bool rho_on = md.rho_out && (!a.ctl || a.ctl->density_on);
  const int64_t tiles = ceil_div(a.n, P);

  // ---- stage weights (bf16x3, rows = output unit), transforms, |det A| ----
  for (int e = tid; e < 64 * 16; e += NTA) {
    const int r = e >> 4, c0 = (e & 15) * 8;
    umma::store_chunk3(sm + OFF_W1, PLW1, r, c0, 64, md.w1 + r * FE + c0);
  }
  for (int e = tid; e < 64 * 8; e += NTA) {
    const int r = e >> 3, c0 = (e & 7) * 8;
    umma::store_chunk3(sm + OFF_W2, PLW2, r, c0, 64, md.w2 + r * HID + c0);
  }
  for (int e = tid; e < 64 * 12; e += NTA) sTF[e] = md.tf[16 * (e / 12) + (e % 12)];
  if (tid < HID) sW3[tid] = md.w3[tid];
  if (rho_on && tid < md.M) {  // |det A| in f64, as density.py:72-80
    const float* t = md.tf + 16 * tid;
    const double c0 = double(t[5]) * t[10] - double(t[6]) * t[9], c1 = double(t[6]) * t[8] - double(t[4]) * t[10],
                 c2 = double(t[4]) * t[9] - double(t[5]) * t[8];
    sDET[tid] = float(fabs(double(t[0]) * c0 + double(t[1]) * c1 + double(t[2]) * c2));
  }
  if (warp == 0) umma::tmem_alloc(tm_slot, TMEM_COLS);
  if (tid == 0) {
    for (int g = 0; g < NG; ++g) {
      umma::mbar_init(bars + 8 * g + B_H1, 4);    // the four epilogue warps
      umma::mbar_init(bars + 8 * g + B_DZ2, 4);
      umma::mbar_init(bars + 8 * g + B_DZ1, 4);
      for (int k = B_Z1; k <= B_GF; ++k) umma::mbar_init(bars + 8 * g + k, 1);  // tcgen05.commit
    }
    umma::fence_mbar_init();
  }
  umma::fence_async_smem();
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tmem = *tm_slot;
  // zero the TMEM-resident weight-gradient sums (warps 0-3 cover the four lane quarters)
  if (warp < 4) {
    uint32_t z[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) z[i] = 0u;
#pragma unroll 1
    for (int c = 0; c < 192; c += 16) umma::tmem_st16(tmem + (uint32_t(32 * warp) << 16) + TC_DW1 + c, z);
    umma::tmem_st_wait();
  }
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t base16 = umma::smem_u32(sm) >> 4;

  double loss = 0.0, srho = 0.0;
  float dw3_acc[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) dw3_acc[c] = 0.f;
  int my_g = -1, my_q = 0;

  {
    // ================= worker groups =================
    const int g = warp / GW, w = warp % GW;
    const int q = w & 3, wq = w >> 2;  // TMEM lane quarter; column half in the epilogues
    my_g = g;
    my_q = q;
    const bool epi = q < 2;            // accumulator rows 0..31 (the tile) live in quarters 0, 1
    uint64_t* gb = bars + 8 * g;
    unsigned char* F = sm + OFF_GRP + g * G_BYTES + G_F;
    unsigned char* H1 = sm + OFF_GRP + g * G_BYTES + G_H1;
    unsigned char* DZ = sm + OFF_GRP + g * G_BYTES + G_DZ;
    float* GF = reinterpret_cast<float*>(F);
    const uint32_t lane_base = uint32_t(32 * q) << 16;
    const uint32_t TA = tmem + 128 * g;
    // M=64 accumulator read with the 16x256b shape: thread t owns rows r0 = 16 q + t/4 and r0 + 8,
    // columns col0 + 8 r + ec (+1) of each 8-column repetition r
    const int r0 = 16 * q + (lane >> 2), r1 = r0 + 8, ec = 2 * (lane & 3);
    const float coef = __fmul_rn(float(2.0 / double(a.n)), md.span);
    const bool issuer = w == ISSUER && lane == 0;
    const uint32_t gbase = OFF_GRP + g * G_BYTES;
    const uint32_t id_kk = umma::idesc_bf16(64, 64, false, false);
    const uint32_t id_kmn = umma::idesc_bf16(64, 64, false, true);
    const uint32_t id_kmn128 = umma::idesc_bf16(64, 128, false, true);
    const uint32_t id_mm = umma::idesc_bf16(64, 64, true, true);
    const uint32_t id_mm128 = umma::idesc_bf16(64, 128, true, true);
    // the group's products, stage s: 0 z1 = F W1^T | 1 z2 = h1 W2^T | 2 dz1 = dz2 W2, dW2 += dz2^T h1 |
    // 3 gF = dz1 W1 (N=128 over acc A|B), dW1 += dz1^T F; each committed to its mbarrier
    auto issue = [&](int stage) {
      umma::fence_after_sync();
      const uint32_t TB = TA + 64;
      if (stage == 0) {
        for (int kk = 0; kk < FE / 16; ++kk)
#pragma unroll
          for (int q6 = 0; q6 < 6; ++q6)
            umma::mma_bf16_c(TA, base16, umma::kmajor_c(gbase + G_F + kPA(q6) * PLF, P, kk),
                             umma::kmajor_c(OFF_W1 + kPB(q6) * PLW1, 64, kk), id_kk, (kk | q6) ? 1u : 0u);
        umma::commit(gb + B_Z1);
      } else if (stage == 1) {
        for (int kk = 0; kk < HID / 16; ++kk)
#pragma unroll
          for (int q6 = 0; q6 < 6; ++q6)
            umma::mma_bf16_c(TB, base16, umma::kmajor_c(gbase + G_H1 + kPA(q6) * PLH, P, kk),
                             umma::kmajor_c(OFF_W2 + kPB(q6) * PLW2, 64, kk), id_kk, (kk | q6) ? 1u : 0u);
        umma::commit(gb + B_Z2);
      } else if (stage == 2) {
        for (int kk = 0; kk < HID / 16; ++kk)
#pragma unroll
          for (int q3 = 0; q3 < 3; ++q3)
            umma::mma_bf16_c(TA, base16, umma::kmajor_c(gbase + G_DZ + kPA(q3) * PLH, P, kk),
                             umma::mnmajor16_c(OFF_W2 + kPB(q3) * PLW2, 64, kk), id_kmn, (kk | q3) ? 1u : 0u);
        for (int kk = 0; kk < P / 16; ++kk)
#pragma unroll
          for (int q3 = 0; q3 < 3; ++q3)
            umma::mma_bf16_c(tmem + TC_DW2, base16, umma::mnmajor16_c(gbase + G_DZ + kPA(q3) * PLH, P, kk),
                             umma::mnmajor16_c(gbase + G_H1 + kPB(q3) * PLH, P, kk), id_mm, 1u);
        umma::commit(gb + B_D1);
      } else {
        for (int kk = 0; kk < HID / 16; ++kk)
#pragma unroll
          for (int q3 = 0; q3 < 3; ++q3)
            umma::mma_bf16_c(TA, base16, umma::kmajor_c(gbase + G_DZ + kPA(q3) * PLH, P, kk),
                             umma::mnmajor16_c(OFF_W1 + kPB(q3) * PLW1, 64, kk), id_kmn128, (kk | q3) ? 1u : 0u);
        for (int kk = 0; kk < P / 16; ++kk)
#pragma unroll
          for (int q3 = 0; q3 < 3; ++q3)
            umma::mma_bf16_c(tmem + TC_DW1, base16, umma::mnmajor16_c(gbase + G_DZ + kPA(q3) * PLH, P, kk),
                             umma::mnmajor16_c(gbase + G_F + kPB(q3) * PLF, P, kk), id_mm128, 1u);
        umma::commit(gb + B_GF);
      }
    };
    const int64_t ntile = group_tiles(tiles, g);
    uint32_t ph = 0;
    const float* tfw = sTF + 12 * (8 * w);  // this warp's grids 8w .. 8w + 7
    // this lane's point of the first tile
    float X0 = 0.f, X1 = 0.f, X2 = 0.f;
    {
      const int64_t i = (2 * int64_t(blockIdx.x) + g) * P + lane;
      if (ntile > 0 && i < a.n) {
        X0 = __ldg(a.coords + 3 * i);
        X1 = __ldg(a.coords + 3 * i + 1);
        X2 = __ldg(a.coords + 3 * i + 2);
      }
    }
    for (int64_t k = 0; k < ntile; ++k) {
      const int64_t tile = 2 * int64_t(blockIdx.x) + g + k * 2 * int64_t(gridDim.x);
      const int cnt = int(min64(P, a.n - tile * P));
      // next tile's point: loaded now, consumed after the scatter
      float N0 = 0.f, N1 = 0.f, N2 = 0.f;
      {
        const int64_t i = (tile + 2 * int64_t(gridDim.x)) * P + lane;
        if (k + 1 < ntile && i < a.n) {
          N0 = __ldg(a.coords + 3 * i);
          N1 = __ldg(a.coords + 3 * i + 1);
          N2 = __ldg(a.coords + 3 * i + 2);
        }
      }
      // ---- encode: point `lane`, grids 8w .. 8w + 7 (two per pass, packed) ----
      {
        float fv[16];
        float racc = 0.f;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int m0 = 8 * w + 2 * jj;
          const float* ta = tfw + 24 * jj;
          const float* tb = ta + 12;
          const float2 l0 = local_axis_g2(X0, X1, X2, ta, tb);
          const float2 l1 = local_axis_g2(X0, X1, X2, ta + 4, tb + 4);
          const float2 l2 = local_axis_g2(X0, X1, X2, ta + 8, tb + 8);
          if (rho_on) {
            const float2 b = bump_p10x2(l0, l1, l2);
            racc = fmaf(sDET[m0 + 1], b.y, fmaf(sDET[m0], b.x, racc));
          }
          int ix[2], iy[2], iz[2];
          float fx[2], fy[2], fz[2];
          axis_term2(l0, md.W, ix[0], ix[1], fx[0], fx[1]);
          axis_term2(l1, md.H, iy[0], iy[1], fy[0], fy[1]);
          axis_term2(l2, md.D, iz[0], iz[1], fz[0], fz[1]);
          const float la[2][3] = {{l0.x, l1.x, l2.x}, {l0.y, l1.y, l2.y}};
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const bool inside = (fabsf(la[h][0]) <= 1.f) && (fabsf(la[h][1]) <= 1.f) && (fabsf(la[h][2]) <= 1.f);
            const int vb = inside ? (((m0 + h) * md.D + iz[h]) * md.H + iy[h]) * md.W + ix[h] : 0;
            float f0, f1;
            if (md.gridx)
              interp_pairx_f32(md.gridx, md.W, md.H * md.W, vb, fx[h], fy[h], fz[h], f0, f1);
            else
              interp_pair_f32(md.grid, md.W, md.H * md.W, vb, fx[h], fy[h], fz[h], f0, f1);
            fv[4 * jj + 2 * h] = inside ? f0 : 0.f;
            fv[4 * jj + 2 * h + 1] = inside ? f1 : 0.f;
          }
        }
        umma::store_chunk3(F, PLF, lane, 16 * w, P, fv);
        umma::store_chunk3(F, PLF, lane, 16 * w + 8, P, fv + 8);
        if (rho_on) sRHO[(g * GW + w) * P + lane] = racc;
      }
      umma::fence_async_smem();
      umma::fence_before_sync();
      umma::named_sync(1 + g, GT);  // F and the group's rho partials are in place
      if (issuer) issue(0);
      if (rho_on && w == 2) {       // a warp with no epilogue rows sums rho per point, in warp order
        float r = 0.f;
#pragma unroll
        for (int v = 0; v < GW; ++v) r += sRHO[(g * GW + v) * P + lane];
        const int64_t i = tile * P + lane;
        if (lane < cnt) {
          md.rho_out[i] = double(r);
          srho += double(r);
        }
      }
      if (issuer) {  // the rest of the chain as the epilogue warps publish each operand
#pragma unroll 1
        for (int st = 1; st < 4; ++st) {
          umma::mbar_wait(gb + (st == 1 ? B_H1 : (st == 2 ? B_DZ2 : B_DZ1)), ph);
          issue(st);
        }
      }
      __syncwarp();
      uint32_t h1pos = 0;
      if (epi) {
        // ---- epilogue 1: h1 = relu(z1) -> bf16x3; sign bits kept for the dz1 mask ----
        umma::mbar_wait(gb + B_Z1, ph);
        umma::fence_after_sync();
        float v[16];
        umma::tmem_ld_16x256b_x4(TA + lane_base + 32 * wq, v);
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          if (v[e] > 0.f) h1pos |= 1u << e;
          v[e] = fmaxf(v[e], 0.f);
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          umma::store_pair3(H1, PLH, r0, 32 * wq + 8 * r + ec, P, v[4 * r], v[4 * r + 1]);
          umma::store_pair3(H1, PLH, r1, 32 * wq + 8 * r + ec, P, v[4 * r + 2], v[4 * r + 3]);
        }
        umma::fence_async_smem();
        umma::fence_before_sync();
        __syncwarp();
        if (lane == 0) umma::mbar_arrive(gb + B_H1);
        // ---- epilogue 2: h2, head, loss, g = dL/dout, dz2 = [z2 > 0] g w3, dW3 ----
        umma::mbar_wait(gb + B_Z2, ph);
        umma::fence_after_sync();
        umma::tmem_ld_16x256b_x4(TA + 64 + lane_base + 32 * wq, v);
        float part0 = 0.f, part1 = 0.f;
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const float w3 = sW3[32 * wq + 8 * r + ec + j];
            v[4 * r + j] = fmaxf(v[4 * r + j], 0.f);
            v[4 * r + 2 + j] = fmaxf(v[4 * r + 2 + j], 0.f);
            part0 = fmaf(v[4 * r + j], w3, part0);
            part1 = fmaf(v[4 * r + 2 + j], w3, part1);
          }
        part0 += __shfl_xor_sync(0xffffffffu, part0, 1);
        part0 += __shfl_xor_sync(0xffffffffu, part0, 2);
        part1 += __shfl_xor_sync(0xffffffffu, part1, 1);
        part1 += __shfl_xor_sync(0xffffffffu, part1, 2);
        if ((lane & 3) == 0) {
          sHead[(g * 2 + wq) * P + r0] = part0;
          sHead[(g * 2 + wq) * P + r1] = part1;
        }
        umma::named_sync(3 + 2 * g + q, 64);  // the two warps of this quarter (w = q, q + 4)
        float gg[2];
#pragma unroll
        for (int kq = 0; kq < 2; ++kq) {
          const int pr = kq ? r1 : r0;
          gg[kq] = 0.f;
          if (pr < cnt) {
            const float raw = sHead[(g * 2) * P + pr] + sHead[(g * 2 + 1) * P + pr];
            const float y = __fadd_rn(__fmul_rn(raw, md.span), md.vmin);
            const float r = __fsub_rn(y, __ldg(a.targets + tile * P + pr));
            const float sqe = __fmul_rn(r, r);
            if (wq == 0 && (lane & 3) == 0) {  // one writer per point
              a.sq[tile * P + pr] = sqe;
              loss += double(sqe);
            }
            gg[kq] = __fmul_rn(r, coef);
          }
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          float d0[2], d1[2];
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const float w3 = sW3[32 * wq + 8 * r + ec + j];
            const float a0 = v[4 * r + j], a1 = v[4 * r + 2 + j];
            dw3_acc[2 * r + j] = fmaf(gg[1], a1, fmaf(gg[0], a0, dw3_acc[2 * r + j]));
            d0[j] = a0 > 0.f ? __fmul_rn(gg[0], w3) : 0.f;  // g_z2 (optim.py:143-145)
            d1[j] = a1 > 0.f ? __fmul_rn(gg[1], w3) : 0.f;
          }
          umma::store_pair2(DZ, PLH, r0, 32 * wq + 8 * r + ec, P, d0[0], d0[1]);
          umma::store_pair2(DZ, PLH, r1, 32 * wq + 8 * r + ec, P, d1[0], d1[1]);
        }
        umma::fence_async_smem();
        umma::fence_before_sync();
        __syncwarp();
        if (lane == 0) umma::mbar_arrive(gb + B_DZ2);
        // ---- epilogue 3: dz1 *= [h1 > 0] -> bf16 (h, m) over dz2 (consumed by dz1 || dW2) ----
        umma::mbar_wait(gb + B_D1, ph);
        umma::fence_after_sync();
        umma::tmem_ld_16x256b_x4(TA + lane_base + 32 * wq, v);
#pragma unroll
        for (int e = 0; e < 16; ++e)
          if (!((h1pos >> e) & 1u)) v[e] = 0.f;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          umma::store_pair2(DZ, PLH, r0, 32 * wq + 8 * r + ec, P, v[4 * r], v[4 * r + 1]);
          umma::store_pair2(DZ, PLH, r1, 32 * wq + 8 * r + ec, P, v[4 * r + 2], v[4 * r + 3]);
        }
        umma::fence_async_smem();
        umma::fence_before_sync();
        __syncwarp();
        if (lane == 0) umma::mbar_arrive(gb + B_DZ1);
        // ---- epilogue 4: gF (acc A|B, 64 columns per warp) -> f32 [32][128] over F ----
        umma::mbar_wait(gb + B_GF, ph);
        umma::fence_after_sync();
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          umma::tmem_ld_16x256b_x4(TA + lane_base + 64 * wq + 32 * half, v);
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int c = 64 * wq + 32 * half + 8 * r + ec;
            *reinterpret_cast<float2*>(GF + gf_idx(r0, c)) = make_float2(v[4 * r], v[4 * r + 1]);
            *reinterpret_cast<float2*>(GF + gf_idx(r1, c)) = make_float2(v[4 * r + 2], v[4 * r + 3]);
          }
        }
        umma::fence_before_sync();
      }
      umma::named_sync(1 + g, GT);  // gF complete
      umma::fence_after_sync();
      // ---- scatter: point `lane`, grids 8w .. 8w + 7, cell terms recomputed ----
      {
        float gv[16];
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) {
          const float4 t4 = *reinterpret_cast<const float4*>(GF + gf_idx(lane, 16 * w + 4 * c4));
          gv[4 * c4] = t4.x;
          gv[4 * c4 + 1] = t4.y;
          gv[4 * c4 + 2] = t4.z;
          gv[4 * c4 + 3] = t4.w;
        }
        const bool live = lane < cnt;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int m0 = 8 * w + 2 * jj;
          const float* ta = tfw + 24 * jj;
          const float* tb = ta + 12;
          const float2 l0 = local_axis_g2(X0, X1, X2, ta, tb);
          const float2 l1 = local_axis_g2(X0, X1, X2, ta + 4, tb + 4);
          const float2 l2 = local_axis_g2(X0, X1, X2, ta + 8, tb + 8);
          int ix[2], iy[2], iz[2];
          float fx[2], fy[2], fz[2];
          axis_term2(l0, md.W, ix[0], ix[1], fx[0], fx[1]);
          axis_term2(l1, md.H, iy[0], iy[1], fy[0], fy[1]);
          axis_term2(l2, md.D, iz[0], iz[1], fz[0], fz[1]);
          const float la[2][3] = {{l0.x, l1.x, l2.x}, {l0.y, l1.y, l2.y}};
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const bool valid =
                live && (fabsf(la[h][0]) <= 1.f) && (fabsf(la[h][1]) <= 1.f) && (fabsf(la[h][2]) <= 1.f);
            const int vb = valid ? (((m0 + h) * md.D + iz[h]) * md.H + iy[h]) * md.W + ix[h] : -1;
            const float g0 = valid ? gv[4 * jj + 2 * h] : 0.f, g1 = valid ? gv[4 * jj + 2 * h + 1] : 0.f;
            scatter_vertex_warp_gather<FX>(md, a.dgrid, valid, vb, fx[h], fy[h], fz[h], g0, g1);
          }
        }
      }
      umma::named_sync(1 + g, GT);  // every warp has read gF before the next encode overwrites F
      X0 = N0;
      X1 = N1;
      X2 = N2;
      ph ^= 1u;
    }
  }

  // ---- flush per-CTA partials: [dW1 (64x128) | dW2 (64x64) | dW3 (64)] from TMEM ----
  // dW3: the 8 lanes sharing lane & 3 hold the same columns; one slot per (group, quarter)
  if (my_g >= 0 && my_q < 2) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      float v = dw3_acc[c];
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      const int wq = (warp % GW) >> 2;
      if (lane < 4) sDW3[(my_g * 2 + my_q) * HID + 32 * wq + 8 * (c >> 1) + 2 * lane + (c & 1)] = v;
    }
  }
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  float* dst = a.part_dw + int64_t(blockIdx.x) * (HID * FE + HID * HID + HID);
  if (warp < NWK) {  // 16 warps: quarter = warp & 3, 16-column slice (warp >> 2)
    const int q = warp & 3, c0 = 16 * (warp >> 2);
    const int p0 = 16 * q + (lane >> 2), p1 = p0 + 8, ec = 2 * (lane & 3);
    const uint32_t lb = uint32_t(32 * q) << 16;
    float v[16];
    umma::tmem_ld_16x256b_x4(tmem + TC_DW1 + lb + 2 * c0, v);  // dW1 rows i = p0 / p1, 32 columns
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int k = 2 * c0 + 8 * r + ec;
      dst[p0 * FE + k] = v[4 * r];
      dst[p0 * FE + k + 1] = v[4 * r + 1];
      dst[p1 * FE + k] = v[4 * r + 2];
      dst[p1 * FE + k + 1] = v[4 * r + 3];
    }
    umma::tmem_ld_16x256b_x2(tmem + TC_DW2 + lb + c0, v);  // dW2 rows j = p0 / p1, 16 columns
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int i = c0 + 8 * r + ec;
      dst[HID * FE + p0 * HID + i] = v[4 * r];
      dst[HID * FE + p0 * HID + i + 1] = v[4 * r + 1];
      dst[HID * FE + p1 * HID + i] = v[4 * r + 2];
      dst[HID * FE + p1 * HID + i + 1] = v[4 * r + 3];
    }
  }
  const double bl = block_sum(loss, red);  // contains __syncthreads
  if (rho_on) {
    const double br = block_sum(srho, red);
    if (tid == 0) {  // the rho pass's (sum rho, sum sq_err) partials, one pair per CTA
      md.rho_part[2 * blockIdx.x] = br;
      md.rho_part[2 * blockIdx.x + 1] = bl;
    }
  }
  if (tid < HID) {  // fixed-order sum over (group, quarter): run-to-run deterministic
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < NG * 2; ++k) s += sDW3[k * HID + tid];
    dst[HID * FE + HID * HID + tid] = s;
  }
  if (tid == 0) a.part_loss[blockIdx.x] = bl;
  umma::fence_before_sync();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tmem, TMEM_COLS);
}

}  // namespace pp

bool recon_pp_selected() {
  static const bool on = [] {
    const char* e = getenv("APMG_RECON");
    return e && e[0] == 'p';
  }();
  return on;
}

int launch_recon_pp(const ModelDev<float>& md, int64_t n, const float* coords, const float* targets, float* sq,
                    float* dgrid, float* part_dw, double* part_loss, int grid, const TrainCtl* ctl,
                    cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    APMG_CUDA_TRY(cudaFuncSetAttribute(pp::k_recon_pp<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(pp::SMEM_BYTES)));
    APMG_CUDA_TRY(cudaFuncSetAttribute(pp::k_recon_pp<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(pp::SMEM_BYTES)));
    attr = true;
  }
  pp::Args a{md, n, coords, targets, sq, dgrid, part_dw, part_loss, ctl};
  if (md.dgrid_fx)
    APMG_LAUNCH("recon_fwd_bwd_tc", pp::k_recon_pp<true>, grid, pp::NTA, pp::SMEM_BYTES, st, a);
  else
    APMG_LAUNCH("recon_fwd_bwd_tc", pp::k_recon_pp<false>, grid, pp::NTA, pp::SMEM_BYTES, st, a);
  return APMG_OK;
}

}  // namespace apmg
