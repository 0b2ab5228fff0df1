// Fused reconstruction step (optim.py:102-155) for the flagship shape (float32, 64 grids x
// 2 channels -> 128 features, 64 hidden), every product on the 5th-gen tensor core with
// bf16x3 operands (x = h + m + l, 8+8+8 significant bits; tcgen05.mma kind::f16, f32
// accumulate).  16-bit operands are accepted K-major and MN-major from the same CM buffer,
// so the transposed products of the backward read the forward's buffers directly.
//
// One persistent CTA (16 warps) per SM; a 64-point tile per loop iteration:
//   encode      (point, grid) pairs -> features F (bf16x3), cell terms cached in TMEM
//   z1 = F W1^T                         M=64 N=64  K=128, 6 products (f32-level accuracy)
//   h1 = relu(z1) -> bf16x3, sign bitmap
//   z2 = h1 W2^T                        M=64 N=64  K=64, 6 products
//   head/loss, g = dL/dout, dz2 = [z2>0] g w3 -> bf16x3
//   dz1 = dz2 W2      (B = W2 MN-major) M=64 N=64  K=64, 3 products (hh, hm, mh)
//   dW2 += dz2^T h1   (A, B MN-major)   M=64 N=64  K=64, 3 products, TMEM-resident sum
//   dz1 *= [h1 > 0] -> bf16x3
//   gF = dz1 W1       (B = W1 MN-major) M=64 N=128 K=64, 3 products
//   dW1 += dz1^T F    (A, B MN-major)   M=64 N=128 K=64, 3 products, TMEM-resident sum
//   scatter     gF -> x-pair grid gradients (warp-aggregated float4 RED), interleaved
//               with the encode of the next tile
// The backward products keep ~2^-16 relative accuracy per term (gradient gate 1e-3); the
// forward keeps the f32-level 6-product split (forward / loss gates).
//
// Shared memory (~199 KB): W1 | W2 | F | h1 | dz2 | dz1 (bf16x3, 16-bit CM layout) | small;
// gF (f32, swizzled) reuses [h1 | dz2] once dW2 / dz1 have consumed them.  Tensor memory:
// acc A (z1, then dz1) | acc B (z2) -- gF spans both -- | dW1 | dW2 | per-thread cell cache.
#include "kernels.cuh"
#include "umma.cuh"

namespace apmg {
namespace tc16 {

constexpr int P = 64;
constexpr int NW = 16;
constexpr int NT = 32 * NW;
constexpr int WQ = NW / 4;
constexpr int EPC = 64 / WQ;  // 16
constexpr int GPW = 64 / NW;  // 4
constexpr int FE = 128;
constexpr int HID = 64;

constexpr uint32_t PL64x128 = 64 * 128 * 2, PL64x64 = 64 * 64 * 2;
constexpr uint32_t OFF_W1 = 0;                          // [64 i][128 k] x3
constexpr uint32_t OFF_W2 = OFF_W1 + 3 * PL64x128;      // [64 j][64 i] x3
constexpr uint32_t OFF_F = OFF_W2 + 3 * PL64x64;        // [64 p][128 k] x3
constexpr uint32_t OFF_H1 = OFF_F + 3 * PL64x128;       // [64 p][64 i] x3
constexpr uint32_t OFF_DZ2 = OFF_H1 + 3 * PL64x64;      // [64 p][64 j] x2 (the backward products use h, m)
#ifndef TC16_DZ1_ALIAS
#define TC16_DZ1_ALIAS 1
#endif
// dz1 reuses h1's buffer: h1's last readers (z2, dW2) complete before the dz1 epilogue writes it,
// and the next h1 is written after the gF || dW1 products have read dz1 -- the 16 KB go to L1,
// which holds the encoder's gather reuse (the kernel is bound by L2 requests per SM)
constexpr uint32_t OFF_DZ1 = TC16_DZ1_ALIAS ? OFF_H1 : OFF_DZ2 + 2 * PL64x64;  // [64 p][64 i] x2
constexpr uint32_t OFF_GF = OFF_DZ2 + (TC16_DZ1_ALIAS ? 2 : 4) * PL64x64;  // f32 [64][128]: lives until the next tile's gF
constexpr uint32_t OFF_X = OFF_GF + P * FE * 4;         // [2][P][3]
constexpr uint32_t OFF_T = OFF_X + 2 * P * 3 * 4;       // [2][P]
constexpr uint32_t OFF_HEAD = OFF_T + 2 * P * 4;        // [WQ][P] partial heads per lane-quarter warp
constexpr uint32_t OFF_DW3 = OFF_HEAD + WQ * P * 4;     // [4 quarters][64]: dW3 per lane quarter, summed in order
constexpr uint32_t OFF_RED = OFF_DW3 + 4 * HID * 4;     // [32] doubles
constexpr uint32_t OFF_BAR = OFF_RED + 32 * 8;
constexpr uint32_t OFF_TM = OFF_BAR + 16;               // [bar | bar_dw1]
constexpr uint32_t OFF_TF = (OFF_TM + 8 + 15) & ~15u;   // [64][12], 16-B aligned (3 LDS.128 per grid)
constexpr uint32_t OFF_W3 = OFF_TF + 64 * 12 * 4;       // [64]
constexpr uint32_t OFF_DET = OFF_W3 + 64 * 4;          // [64] |det A| (fused density)
constexpr uint32_t OFF_RHO = OFF_DET + 64 * 4;         // [NW][P] per-warp partial rho (fused density)
constexpr uint32_t SMEM_BYTES = OFF_RHO + NW * P * 4;
static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");

constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t TC_A = 0, TC_B = 64, TC_DW1 = 128, TC_DW2 = 256, TC_CACHE = 320;
// cell cache: 3 words per (grid, point) pair (base vertex, three 21-bit fractions), 12 columns per
// encode group, two groups per warp, four warps per lane quarter = 96 columns per tile; two tiles
// (parity) so the scatter of tile t can run after the encode of tile t+1
constexpr uint32_t CACHE_TILE = 96;
static_assert(TC_CACHE + 2 * CACHE_TILE <= TMEM_COLS, "tensor memory budget");

// where the scatter of tile t runs: SQ_I pairs interleaved with the encode of tile t+1, SQ_Z in the
// wait for its z1, SQ_C in its z2 wait and SQ_E in its dz1 || dW2 wait, the rest in its gF || dW1 wait
#ifndef TC16_SQ_I
#define TC16_SQ_I 0
#define TC16_SQ_Z 2
#define TC16_SQ_C 2
#define TC16_SQ_E 2
#endif
// corner loads issued per batch in the encode before their lerps: 4 (a group's 2 grids x 2 points,
// 16 float4 in flight), 2 (per grid) or 1 (per (grid, point): load -> lerp, the round-1 order)
#ifndef TC16_ENC_BATCH
#define TC16_ENC_BATCH 4
#endif
#ifndef TC16_FWD_Q
#define TC16_FWD_Q 6  // forward products per GEMM: 6 (f32-level) or 3 (hh, hm, mh: ~2^-16)
#endif
constexpr int FWD_Q = TC16_FWD_Q;
// dedicated MMA-issue warp (warp NW, lane 0; warps NW+1..NW+3 idle) instead of thread 0 of worker
// warp 0: an issuing thread blocks while the tensor pipe's queue is full (~24 MMAs of ~51 cycles),
// which made warp 0 the straggler at every barrier of the tile
#ifndef TC16_MMA_WARP
#define TC16_MMA_WARP 1
#endif
constexpr bool kMmaWarp = TC16_MMA_WARP != 0;
// gF and dW1 committed to separate mbarriers: the gF epilogue starts when gF is done while dW1
// (needed only once the next tile overwrites F, and at the flush) still runs
#ifndef TC16_SPLIT_DW1
#define TC16_SPLIT_DW1 1
#endif
constexpr bool kSplitDW1 = TC16_SPLIT_DW1 != 0;
constexpr int NT_LAUNCH = kMmaWarp ? NT + 128 : NT;
// registers: launched at 96 per thread (640 threads); the helper warpgroup releases 64 per thread
// (setmaxnreg.dec) and the workers take them (setmaxnreg.inc blocks until the CTA's pool holds
// them: 16 x (112 - 96) = 4 x (96 - 32))
#ifndef TC16_REG_WORK
#define TC16_REG_WORK 112
#define TC16_REG_HELP 32
#endif
constexpr int REG_WORK = TC16_REG_WORK, REG_HELP = TC16_REG_HELP;
static_assert(!kMmaWarp || NW * (REG_WORK - 96) <= 4 * (96 - REG_HELP), "setmaxnreg.inc would wait forever");
// named barriers: 1 MMA handoff / encode sync (workers + issuing warp), 2-5 lane-quarter head
// exchange, 6 first-half z1 handoff, 7 workers only, 8 end of kernel (all warps)
constexpr int BAR_MMA = 1, BAR_Z1A = 6, BAR_WORK = 7, BAR_END = 8;
constexpr int FWD_PLANES = FWD_Q == 6 ? 3 : 2;
constexpr int SQ_I = TC16_SQ_I, SQ_Z = TC16_SQ_Z, SQ_C = TC16_SQ_C, SQ_E = TC16_SQ_E, SQ = 8;
constexpr int SQ1 = SQ_I + SQ_Z, SQ2 = SQ1 + SQ_C, SQ3 = SQ2 + SQ_E;  // cumulative pair boundaries

// fractions in [0, 1] as 21-bit fixed point (resolution 2^-21; the scatter weights only)
__device__ __forceinline__ void pack_cell(int vbase, float fx, float fy, float fz, uint32_t* w) {
  const uint32_t qx = min(__float2uint_rn(fx * 2097152.f), 2097151u);
  const uint32_t qy = min(__float2uint_rn(fy * 2097152.f), 2097151u);
  const uint32_t qz = min(__float2uint_rn(fz * 2097152.f), 2097151u);
  w[0] = uint32_t(vbase);
  w[1] = qx | (qy << 21);
  w[2] = (qy >> 11) | (qz << 10);
}
__device__ __forceinline__ void unpack_cell(const uint32_t* w, int& vbase, float& fx, float& fy, float& fz) {
  vbase = int(w[0]);
  fx = float(w[1] & 0x1FFFFFu) * 4.76837158203125e-07f;
  fy = float((w[1] >> 21) | ((w[2] & 0x3FFu) << 11)) * 4.76837158203125e-07f;
  fz = float((w[2] >> 10) & 0x1FFFFFu) * 4.76837158203125e-07f;
}

// bf16x3 product q: (A plane, B plane) = hh, hm, mh, hl, lh, mm
__host__ __device__ constexpr int kPA(int q) { return q == 2 ? 1 : (q == 4 ? 2 : (q == 5 ? 1 : 0)); }
__host__ __device__ constexpr int kPB(int q) { return q == 1 ? 1 : (q == 3 ? 2 : (q == 5 ? 1 : 0)); }

// per-phase clock stamps of CTA 0 / thread 0 for the first 16 tiles (APMG_TC_STAMPS=1)
__device__ long long g_tc16_stamp[16][12];
#define TC16_STAMP(k)                                                                   \
  do {                                                                                  \
    if (a.stamps && blockIdx.x == 0 && tid == 0 && it < 16) g_tc16_stamp[it][k] = clock64(); \
    TC16_WSTAMP(k);                                                                     \
  } while (0)
// the same per warp (lane 0 of every warp of CTA 0), with extra points inside the encode and
// before the tensor-core waits (APMG_TC_STAMPS=1; profiling only)
__device__ long long g_tc16_wstamp[16][16][16];
#define TC16_WSTAMP(k)                                                                                          \
  do {                                                                                                          \
    if (a.stamps && blockIdx.x == 0 && (tid & 31) == 0 && it < 16) g_tc16_wstamp[it][tid >> 5][k] = clock64(); \
  } while (0)

// gF [P][128] f32, 8-byte granules XOR-swizzled by row: f(p) maps p & 15 onto the even
// offsets 0..30 so both the row-per-lane float2 scatter reads (16 rows per half warp) and
// the 16x256b epilogue writes (8 rows x 4 column pairs) spread over the banks
__device__ __forceinline__ int gf_idx(int p, int k) { return p * 128 + (k ^ (8 * (p & 3) + 2 * ((p >> 2) & 3))); }

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
  int aggregate;
  int stamps;
};

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

// scatter of pairs [q0, q1) (q = 4 jq + u: grid 2 warp + 32 jq + u / 2, point lane + 32 (u % 2),
// encode_group's order) of a tile whose cell cache starts at tmem_cache
template <bool FX>
__device__ __forceinline__ void scatter_pairs(const ModelDev<float>& md, const Args& a, const float* GF,
                                              uint32_t tmem_cache, int q0, int q1, int cnt, int warp, int lane) {
#ifdef TC16_ABL_NOSCATTER  // timing ablation only: no scatter at all (wrong results)
  return;
#endif
#pragma unroll
  for (int jq = 0; jq < 2; ++jq) {
    if (q1 <= 4 * jq || q0 >= 4 * jq + 4) continue;  // warp-uniform
    uint32_t cache[12];
    umma::tmem_ld12u(tmem_cache + 12 * jq, cache);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int q = 4 * jq + u;
      if (q < q0 || q >= q1) continue;
      const int m = 2 * warp + 32 * jq + (u >> 1), p = lane + 32 * (u & 1);
      int vbase;
      float fx, fy, fz;
      unpack_cell(cache + 3 * u, vbase, fx, fy, fz);
      const bool valid = vbase >= 0 && p < cnt;
      float2 g = *reinterpret_cast<const float2*>(GF + gf_idx(p, 2 * m));  // p < 64: always in the buffer
      if (!valid) g = make_float2(0.f, 0.f);
      if (a.aggregate == 2)
        scatter_vertex_warp_gather<FX>(md, a.dgrid, valid, vbase, fx, fy, fz, g.x, g.y);
      else if (a.aggregate)
        scatter_vertex_warp_agg(md, a.dgrid, valid, vbase, fx, fy, fz, g.x, g.y);
      else if (valid)
        scatter_vertex_f32(md, a.dgrid, vbase, fx, fy, fz, g.x, g.y);
    }
  }
}

__device__ __forceinline__ float ex2_ftz(float v) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}

// flat-top bump exp(-sum_d l_d^20) of density.py:83-103 (p = 10) for two points in f32, the
// arithmetic of k_dens_rho32x2 (l^2 clamped at 4 so the power cannot overflow), both points in
// packed fp32x2 (each half rounded as the scalar operation; no product feeds an add)
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

template <bool FX>  // FX: deterministic training (fixed-point grid gradient)
__global__ void __launch_bounds__(NT_LAUNCH, 1) k_recon_tc16(Args a) {
  extern __shared__ __align__(1024) unsigned char sm[];
  if (a.ctl && a.ctl->skip) return;
  const ModelDev<float>& md = a.md;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int quarter = warp & 3, wq = warp >> 2;
  unsigned char* W1 = sm + OFF_W1;
  unsigned char* W2 = sm + OFF_W2;
  unsigned char* F = sm + OFF_F;
  unsigned char* H1 = sm + OFF_H1;
  unsigned char* DZ2 = sm + OFF_DZ2;
  unsigned char* DZ1 = sm + OFF_DZ1;
  float* GF = reinterpret_cast<float*>(sm + OFF_GF);
  float* sX = reinterpret_cast<float*>(sm + OFF_X);
  float* sT = reinterpret_cast<float*>(sm + OFF_T);
  float* sHead = reinterpret_cast<float*>(sm + OFF_HEAD);
  float* sDW3 = reinterpret_cast<float*>(sm + OFF_DW3);
  double* red = reinterpret_cast<double*>(sm + OFF_RED);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + OFF_BAR);
  uint32_t* tm_slot = reinterpret_cast<uint32_t*>(sm + OFF_TM);
  float* sTF = reinterpret_cast<float*>(sm + OFF_TF);
  float* sW3 = reinterpret_cast<float*>(sm + OFF_W3);
  float* sDET = reinterpret_cast<float*>(sm + OFF_DET);
  float* sRHO = reinterpret_cast<float*>(sm + OFF_RHO);
  const bool rho_on = md.rho_out && (!a.ctl || a.ctl->density_on);

  // ---- stage weights (bf16x3, rows = output unit) ----
  for (int e = tid; e < 64 * 16 && tid < NT; e += NT) {
    const int r = e >> 4, c0 = (e & 15) * 8;
    umma::store_chunk3(W1, PL64x128, r, c0, 64, md.w1 + r * FE + c0);
  }
  for (int e = tid; e < 64 * 8 && tid < NT; e += NT) {
    const int r = e >> 3, c0 = (e & 7) * 8;
    umma::store_chunk3(W2, PL64x64, r, c0, 64, md.w2 + r * HID + c0);
  }
  for (int e = tid; e < 64 * 12 && tid < NT; e += NT) sTF[e] = md.tf[16 * (e / 12) + (e % 12)];
  if (tid < HID) sW3[tid] = md.w3[tid];
  if (rho_on && tid < md.M) {  // |det A| in f64, as density.py:72-80 (stage_transforms32)
    const float* t = md.tf + 16 * tid;
    const double c0 = double(t[5]) * t[10] - double(t[6]) * t[9], c1 = double(t[6]) * t[8] - double(t[4]) * t[10],
                 c2 = double(t[4]) * t[9] - double(t[5]) * t[8];
    sDET[tid] = float(fabs(double(t[0]) * c0 + double(t[1]) * c1 + double(t[2]) * c2));
  }
  if (warp == 0) umma::tmem_alloc(tm_slot, TMEM_COLS);
  if (tid == 0) {
    umma::mbar_init(bar, 1);
    umma::mbar_init(bar + 1, 1);
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
  const uint32_t TA = tmem + TC_A, TB = tmem + TC_B, TDW1 = tmem + TC_DW1, TDW2 = tmem + TC_DW2;
  // cell cache of tile parity b: tmem_cache0 + b * CACHE_TILE (+ 12 per encode group)
  const uint32_t tmem_cache0 = tmem + TC_CACHE + 24 * wq + lane_base;
  // zero the TMEM-resident weight-gradient sums (warps 0-3 cover the four lane quarters)
  if (warp < 4) {
    uint32_t z[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) z[i] = 0u;
#pragma unroll 1
    for (int c = 0; c < 192; c += 16) umma::tmem_st16(tmem + lane_base + TC_DW1 + c, z);
    umma::tmem_st_wait();
  }
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();

  const uint32_t base16 = umma::smem_u32(sm) >> 4;  // descriptors: base16 + compile-time fields
  const uint32_t id_kk = umma::idesc_bf16(64, 64, false, false);      // A, B K-major
  const uint32_t id_kmn = umma::idesc_bf16(64, 64, false, true);      // B MN-major
  const uint32_t id_kmn128 = umma::idesc_bf16(64, 128, false, true);  // B MN-major, N=128
  const uint32_t id_mm = umma::idesc_bf16(64, 64, true, true);        // A, B MN-major
  const uint32_t id_mm128 = umma::idesc_bf16(64, 128, true, true);
  const float coef = __fmul_rn(float(2.0 / double(a.n)), md.span);
  const bool issuer = kMmaWarp ? (warp == NW && lane == 0) : (tid == 0);

  // M=64 accumulators are read with the 16x256b shape: thread t owns rows p0 = 16q + t/4 and
  // p1 = p0 + 8, columns ep_col0 + 8r + ec (+1) of each 8-column repetition r
  const int ep_col0 = EPC * wq;
  const int p0 = 16 * quarter + (lane >> 2), p1 = p0 + 8, ec = 2 * (lane & 3);
  float dw3_acc[4];  // columns ep_col0 + 8r + ec + j, index 2r + j
#pragma unroll
  for (int c = 0; c < 4; ++c) dw3_acc[c] = 0.f;
  double loss = 0.0;
  double srho = 0.0;  // fused density: sum of this CTA's rho
  uint32_t phase = 0;
  uint32_t phase_dw1 = 0;    // bar + 1 (dW1 products of the previous tile)
  bool dw1_pending = false;  // a tile's dW1 has been issued and not yet waited for
  uint32_t h1pos = 0;  // [h1 > 0] bits of this thread's 8 elements (epilogue 1 -> dz1 epilogue)

  // encode of grids 2 warp + 32 jq + {0, 1} for points lane, lane + 32: the two points of a grid
  // share its transform and run in packed fp32x2 arithmetic; the two grids' four features of a
  // point are adjacent in F (one 8-byte store per plane)
  int it = 0;
  // mid(jj): work with no dependence on the gathers (the previous tile's scatter pairs), run
  // between the issue of grid jj's corner loads and their lerps
  auto encode_group = [&](const float* cX, int jq, uint32_t tmem_cache, float2& racc, auto&& mid) {
    const float2 X0 = make_float2(cX[3 * lane], cX[3 * (lane + 32)]);
    const float2 X1 = make_float2(cX[3 * lane + 1], cX[3 * (lane + 32) + 1]);
    const float2 X2 = make_float2(cX[3 * lane + 2], cX[3 * (lane + 32) + 2]);
    uint32_t cache[12];
    uint32_t fw[2][2][3];  // [grid jj][point h][plane]
    int vbs[2][2];            // [jj][h] base vertex (-1 outside)
    float fxs[2][2], fys[2][2], fzs[2][2];
    // cell terms of grid jj for both points (packed fp32x2), the fused density bump
    auto cells = [&](int jj) {
      const int m = 2 * warp + 32 * jq + jj;
      const float4* tf4 = reinterpret_cast<const float4*>(sTF + 12 * m);  // warp-uniform: 3 broadcasts
      const float4 ta = tf4[0], tb = tf4[1], tc = tf4[2];
      const float2 l0 = local_coord2(X0, X1, X2, ta.x, ta.y, ta.z, ta.w);
      const float2 l1 = local_coord2(X0, X1, X2, tb.x, tb.y, tb.z, tb.w);
      const float2 l2 = local_coord2(X0, X1, X2, tc.x, tc.y, tc.z, tc.w);
      if (rho_on) {
#ifdef TC16_ABL_NOBUMP  // timing ablation only: bump 1 (rho stays positive, training stays finite)
        const float2 b = make_float2(1.f, 1.f);
#else
        const float2 b = bump_p10x2(l0, l1, l2);
#endif
        racc = make_float2(fmaf(sDET[m], b.x, racc.x), fmaf(sDET[m], b.y, racc.y));
      }
      int ix[2], iy[2], iz[2];
      axis_term2(l0, md.W, ix[0], ix[1], fxs[jj][0], fxs[jj][1]);
      axis_term2(l1, md.H, iy[0], iy[1], fys[jj][0], fys[jj][1]);
      axis_term2(l2, md.D, iz[0], iz[1], fzs[jj][0], fzs[jj][1]);
      const float la[2][3] = {{l0.x, l1.x, l2.x}, {l0.y, l1.y, l2.y}};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const bool inside = (fabsf(la[h][0]) <= 1.f) && (fabsf(la[h][1]) <= 1.f) && (fabsf(la[h][2]) <= 1.f);
        vbs[jj][h] = inside ? ((m * md.D + iz[h]) * md.H + iy[h]) * md.W + ix[h] : -1;
      }
    };
    // features of (jj, h) from its gathered corners (straight-line: outside pairs gathered cell 0
    // and are zeroed here), cell cache words, bf16x3 split
    auto finish = [&](int jj, int h, const float4* b) {
      const int u = 2 * jj + h;
      const bool use = vbs[jj][h] >= 0;
      float f0, f1;
      lerp_pairx_f32(b, fxs[jj][h], fys[jj][h], fzs[jj][h], f0, f1);
      f0 = use ? f0 : 0.f;
      f1 = use ? f1 : 0.f;
      pack_cell(vbs[jj][h], fxs[jj][h], fys[jj][h], fzs[jj][h], cache + 3 * u);
      umma::split2_bf16x3(f0, f1, fw[jj][h][0], fw[jj][h][1], fw[jj][h][2]);
    };
    if (md.gridq && TC16_ENC_BATCH == 4) {
      // the xy-quad copy: 2 256-bit loads per (grid, point), the group's 8 issued before its lerps
      cells(0);
      cells(1);
      float b[2][2][16];
#pragma unroll
      for (int jj = 0; jj < 2; ++jj)
#pragma unroll
        for (int h = 0; h < 2; ++h) gather_pairq_f32(md.gridq, md.H * md.W, max(vbs[jj][h], 0), b[jj][h]);
      mid(0);
      mid(1);
#pragma unroll
      for (int jj = 0; jj < 2; ++jj)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int u = 2 * jj + h;
          const bool use = vbs[jj][h] >= 0;
          float f0, f1;
          lerp_pairq_f32(b[jj][h], fxs[jj][h], fys[jj][h], fzs[jj][h], f0, f1);
          f0 = use ? f0 : 0.f;
          f1 = use ? f1 : 0.f;
          pack_cell(vbs[jj][h], fxs[jj][h], fys[jj][h], fzs[jj][h], cache + 3 * u);
          umma::split2_bf16x3(f0, f1, fw[jj][h][0], fw[jj][h][1], fw[jj][h][2]);
        }
    } else if (md.gridx && !md.gridq && TC16_ENC_BATCH == 4) {
      // every corner load of the group issued before the first lerp: 16 float4 gathers in flight
      // per thread instead of 4 (the encode waited one L2 round trip per (grid, point))
      cells(0);
      cells(1);
      float4 b[2][2][4];
#pragma unroll
      for (int jj = 0; jj < 2; ++jj)
#pragma unroll
        for (int h = 0; h < 2; ++h) gather_pairx_f32(md.gridx, md.W, md.H * md.W, max(vbs[jj][h], 0), b[jj][h]);
      mid(0);
      mid(1);
#pragma unroll
      for (int jj = 0; jj < 2; ++jj)
#pragma unroll
        for (int h = 0; h < 2; ++h) finish(jj, h, b[jj][h]);
    } else if (md.gridx && !md.gridq && TC16_ENC_BATCH == 2) {
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {
        cells(jj);
        float4 b[2][4];
#pragma unroll
        for (int h = 0; h < 2; ++h) gather_pairx_f32(md.gridx, md.W, md.H * md.W, max(vbs[jj][h], 0), b[h]);
        mid(jj);
#pragma unroll
        for (int h = 0; h < 2; ++h) finish(jj, h, b[h]);
      }
    } else {
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {
        mid(jj);
        cells(jj);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int u = 2 * jj + h;
          const bool use = vbs[jj][h] >= 0;
          const int vb = use ? vbs[jj][h] : 0;
          float f0 = 0.f, f1 = 0.f;
          if (md.gridq)
            interp_pairq_f32(md.gridq, md.H * md.W, vb, fxs[jj][h], fys[jj][h], fzs[jj][h], f0, f1);
          else if (md.gridx)
            interp_pairx_f32(md.gridx, md.W, md.H * md.W, vb, fxs[jj][h], fys[jj][h], fzs[jj][h], f0, f1);
          else
            interp_pair_f32(md.grid, md.W, md.H * md.W, vb, fxs[jj][h], fys[jj][h], fzs[jj][h], f0, f1);
          f0 = use ? f0 : 0.f;
          f1 = use ? f1 : 0.f;
          pack_cell(vbs[jj][h], fxs[jj][h], fys[jj][h], fzs[jj][h], cache + 3 * u);
          umma::split2_bf16x3(f0, f1, fw[jj][h][0], fw[jj][h][1], fw[jj][h][2]);
        }
      }
    }
    if (kSplitDW1 && jq == 0 && dw1_pending) {  // F is the previous tile's dW1 operand until it is done
      umma::mbar_wait(bar + 1, phase_dw1);
      phase_dw1 ^= 1;
      dw1_pending = false;
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t o = umma::cm16_offset(lane + 32 * h, 4 * warp + 64 * jq, 64);
#pragma unroll
      for (int pl = 0; pl < FWD_PLANES; ++pl)
        *reinterpret_cast<uint2*>(F + pl * PL64x128 + o) = make_uint2(fw[0][h][pl], fw[1][h][pl]);
    }
    umma::tmem_st8(tmem_cache + 12 * jq, cache);
    umma::tmem_st4(tmem_cache + 12 * jq + 8, cache + 8);
  };
  // z1 = F W1^T over K-steps [k0, k1) (K = 16 each), committed when `last`
  auto issue_z1 = [&](int k0, int k1, bool last) {
    if (!issuer) return;
    umma::fence_after_sync();
#pragma unroll 1
    for (int kk = k0; kk < k1; ++kk)
#pragma unroll
      for (int q = 0; q < FWD_Q; ++q)
        umma::mma_bf16_c(TA, base16, umma::kmajor_c(OFF_F + kPA(q) * PL64x128, 64, kk),
                         umma::kmajor_c(OFF_W1 + kPB(q) * PL64x128, 64, kk), id_kk, (kk | q) ? 1u : 0u);
    if (last) umma::commit(bar);
  };
  // z2 = h1 W2^T
  auto issue_z2 = [&]() {
    if (!issuer) return;
    umma::fence_after_sync();
#pragma unroll 1
    for (int kk = 0; kk < HID / 16; ++kk)
#pragma unroll
      for (int q = 0; q < FWD_Q; ++q)
        umma::mma_bf16_c(TB, base16, umma::kmajor_c(OFF_H1 + kPA(q) * PL64x64, 64, kk),
                         umma::kmajor_c(OFF_W2 + kPB(q) * PL64x64, 64, kk), id_kk, (kk | q) ? 1u : 0u);
    umma::commit(bar);
  };
  // dz1 = dz2 W2 (-> acc A), dW2 += dz2^T h1 (-> TMEM sum)
  auto issue_dz1_dw2 = [&]() {
    if (!issuer) return;
    umma::fence_after_sync();
#pragma unroll 1
    for (int kk = 0; kk < HID / 16; ++kk)
#pragma unroll
      for (int q = 0; q < 3; ++q)
        umma::mma_bf16_c(TA, base16, umma::kmajor_c(OFF_DZ2 + kPA(q) * PL64x64, 64, kk),
                         umma::mnmajor16_c(OFF_W2 + kPB(q) * PL64x64, 64, kk), id_kmn, (kk | q) ? 1u : 0u);
#pragma unroll 1
    for (int kk = 0; kk < P / 16; ++kk)
#pragma unroll
      for (int q = 0; q < 3; ++q)
        umma::mma_bf16_c(TDW2, base16, umma::mnmajor16_c(OFF_DZ2 + kPA(q) * PL64x64, 64, kk),
                         umma::mnmajor16_c(OFF_H1 + kPB(q) * PL64x64, 64, kk), id_mm, 1u);
    umma::commit(bar);
  };
  // gF = dz1 W1 (-> acc A|B, N=128), dW1 += dz1^T F (-> TMEM sum)
  auto issue_gf_dw1 = [&]() {
    if (!issuer) return;
    umma::fence_after_sync();
#pragma unroll 1
    for (int kk = 0; kk < HID / 16; ++kk)
#pragma unroll
      for (int q = 0; q < 3; ++q)
        umma::mma_bf16_c(TA, base16, umma::kmajor_c(OFF_DZ1 + kPA(q) * PL64x64, 64, kk),
                         umma::mnmajor16_c(OFF_W1 + kPB(q) * PL64x128, 64, kk), id_kmn128, (kk | q) ? 1u : 0u);
    if constexpr (kSplitDW1) umma::commit(bar);  // the gF epilogue waits for gF only
#pragma unroll 1
    for (int kk = 0; kk < P / 16; ++kk)
#pragma unroll
      for (int q = 0; q < 3; ++q)
        umma::mma_bf16_c(TDW1, base16, umma::mnmajor16_c(OFF_DZ1 + kPA(q) * PL64x64, 64, kk),
                         umma::mnmajor16_c(OFF_F + kPB(q) * PL64x128, 64, kk), id_mm128, 1u);
    umma::commit(kSplitDW1 ? bar + 1 : bar);  // dW1: before the next tile's F stores / the flush
  };
  // operands of the next products are in shared memory: release the issuing thread (the
  // workers arrive and go on; without the MMA warp, warp 0 waits and issues)
  auto handoff = [&](int id) {
    if constexpr (kMmaWarp) {
      umma::named_arrive(id, NT + 32);
    } else {
      if (warp == 0) umma::named_sync(id, NT); else umma::named_arrive(id, NT);
    }
  };
  auto worker_sync = [&]() {
    if constexpr (kMmaWarp) umma::named_sync(BAR_WORK, NT); else __syncthreads();
  };
  // encode of a tile into cache buffer `cache_enc`, with pairs [0, SQ_I) of the previous tile's
  // scatter (cache buffer `cache_sc`, scatter_cnt points; < 0: none) interleaved group by group
  auto encode_tile = [&](const float* cX, uint32_t cache_enc, uint32_t cache_sc, int scatter_cnt,
                         int64_t prefetch_tile, int prefetch_slot) {
    // the tile after next: its coordinates / targets are fetched now (registers) and stored to
    // shared memory after the encode, so the global-load latency hides behind it
    float pf[4] = {0.f, 0.f, 0.f, 0.f};
    float2 racc = make_float2(0.f, 0.f);
    const bool pf_on = prefetch_tile < tiles && tid < P;
    if (pf_on) {
      const int64_t i = prefetch_tile * P + tid;
      if (i < a.n) {
        pf[0] = __ldg(a.coords + 3 * i);
        pf[1] = __ldg(a.coords + 3 * i + 1);
        pf[2] = __ldg(a.coords + 3 * i + 2);
        pf[3] = __ldg(a.targets + i);
      }
    }
#pragma unroll
    for (int jq = 0; jq < GPW / 2; ++jq) {
      // pairs [SQ_I (2 jq + jj) / 4, SQ_I (2 jq + jj + 1) / 4) of the previous tile's scatter run while
      // grid jj's gathers are in flight
      encode_group(cX, jq, cache_enc, racc, [&](int jj) {
        if (SQ_I > 0 && scatter_cnt >= 0)
          scatter_pairs<FX>(md, a, GF, cache_sc, SQ_I * (2 * jq + jj) / 4, SQ_I * (2 * jq + jj + 1) / 4, scatter_cnt,
                            warp, lane);
      });
      TC16_WSTAMP(9 + 2 * jq);
      if (jq == 0) {
        // features k < 64 (grids 0-31) complete: first half of z1.  Only the issuing warp waits
        // for the others; they signal the named barrier and carry on with group 1
        umma::fence_async_smem();
        handoff(BAR_Z1A);
        if constexpr (!kMmaWarp) issue_z1(0, FE / 32, false);
        TC16_WSTAMP(10);
      }
    }
    umma::tmem_st_wait();
    if (rho_on) {  // this warp's 4 grids; summed over the warps in order after the barrier
      sRHO[warp * P + lane] = racc.x;
      sRHO[warp * P + lane + 32] = racc.y;
    }
    if (pf_on) {
      float* dX = sX + (prefetch_slot & 1) * 3 * P;
      dX[3 * tid] = pf[0];
      dX[3 * tid + 1] = pf[1];
      dX[3 * tid + 2] = pf[2];
      sT[(prefetch_slot & 1) * P + tid] = pf[3];
    }
    umma::fence_async_smem();
    umma::fence_before_sync();
    // F complete; every warp's scatter of the previous tile has read gF (with the MMA warp: a
    // barrier of the workers and the issuing warp, which then issues the second half of z1)
    if constexpr (kMmaWarp) umma::named_sync(BAR_MMA, NT + 32); else __syncthreads();
    TC16_WSTAMP(12);
    if constexpr (!kMmaWarp) issue_z1(FE / 32, FE / 16, true);
  };

  if constexpr (kMmaWarp) {
    if (warp >= NW) {
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(REG_HELP));
      if (warp == NW) {  // the issuing warp: the workers' handoffs, in their order
        if (int64_t(blockIdx.x) < tiles) {
          umma::named_sync(BAR_Z1A, NT + 32);
          issue_z1(0, FE / 32, false);
          umma::named_sync(BAR_MMA, NT + 32);
          issue_z1(FE / 32, FE / 16, true);
        }
        for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
          umma::named_sync(BAR_MMA, NT + 32);
          issue_z2();
          umma::named_sync(BAR_MMA, NT + 32);
          issue_dz1_dw2();
          umma::named_sync(BAR_MMA, NT + 32);
          issue_gf_dw1();
          if (tile + gridDim.x < tiles) {
            umma::named_sync(BAR_Z1A, NT + 32);
            issue_z1(0, FE / 32, false);
            umma::named_sync(BAR_MMA, NT + 32);
            issue_z1(FE / 32, FE / 16, true);
          }
        }
      }
      umma::named_sync(BAR_END, NT_LAUNCH);  // the workers' final barrier (TMEM dealloc after it)
      return;
    }
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(REG_WORK));
  }
  if (int64_t(blockIdx.x) < tiles) encode_tile(sX, tmem_cache0, tmem_cache0, -1, int64_t(blockIdx.x) + gridDim.x, 1);
  int cnt_prev = -1;  // the previous tile's scatter pairs [SQ_I, SQ) run in this tile's tensor-core waits
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++it) {
    const int cnt = int(min64(P, a.n - tile * P));
    const float* cT = sT + (it & 1) * P;
    const uint32_t cache_cur = tmem_cache0 + (it & 1) * CACHE_TILE, cache_prev = tmem_cache0 + ((it + 1) & 1) * CACHE_TILE;
    TC16_STAMP(0);
    if (cnt_prev >= 0) scatter_pairs<FX>(md, a, GF, cache_prev, SQ_I, SQ1, cnt_prev, warp, lane);
    umma::mbar_wait(bar, phase);
    phase ^= 1;
    umma::fence_after_sync();
    TC16_STAMP(1);
    if (rho_on && tid >= NT - P) {  // rho of this tile's points: the 16 warp partials in order
      const int pt = tid - (NT - P);
      float r = 0.f;
#pragma unroll
      for (int w = 0; w < NW; ++w) r += sRHO[w * P + pt];
      const int64_t i = tile * P + pt;
      if (i < a.n) {
        md.rho_out[i] = double(r);
        srho += double(r);
      }
    }
    // ---- epilogue 1: h1 = relu(z1) -> bf16x3; sign bits kept in a register ----
    {
      float v[8];
      umma::tmem_ld_16x256b_x2(TA + lane_base + ep_col0, v);
      h1pos = 0;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        if (v[e] > 0.f) h1pos |= 1u << e;
        v[e] = fmaxf(v[e], 0.f);
      }
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        if constexpr (FWD_PLANES == 3) {
          umma::store_pair3(H1, PL64x64, p0, ep_col0 + 8 * r + ec, 64, v[4 * r], v[4 * r + 1]);
          umma::store_pair3(H1, PL64x64, p1, ep_col0 + 8 * r + ec, 64, v[4 * r + 2], v[4 * r + 3]);
        } else {
          umma::store_pair2(H1, PL64x64, p0, ep_col0 + 8 * r + ec, 64, v[4 * r], v[4 * r + 1]);
          umma::store_pair2(H1, PL64x64, p1, ep_col0 + 8 * r + ec, 64, v[4 * r + 2], v[4 * r + 3]);
        }
      }
    }
    umma::fence_async_smem();
    umma::fence_before_sync();
    // only the issuing warp waits for the stores; the others go on to their share of the
    // previous tile's scatter
    handoff(BAR_MMA);
    umma::fence_after_sync();
    TC16_STAMP(2);
    // ---- z2 = h1 W2^T ----
    if constexpr (!kMmaWarp) issue_z2();
    if (cnt_prev >= 0) scatter_pairs<FX>(md, a, GF, cache_prev, SQ1, SQ2, cnt_prev, warp, lane);
    TC16_WSTAMP(13);
    umma::mbar_wait(bar, phase);
    phase ^= 1;
    umma::fence_after_sync();
    TC16_STAMP(3);
    // ---- epilogue 2: h2, head, loss, g, dz2 = [z2 > 0] g w3, dW3 ----
    float h2v[8];
    umma::tmem_ld_16x256b_x2(TB + lane_base + ep_col0, h2v);
    {
      float part0 = 0.f, part1 = 0.f;
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const float w = sW3[ep_col0 + 8 * r + ec + j];
          h2v[4 * r + j] = fmaxf(h2v[4 * r + j], 0.f);
          h2v[4 * r + 2 + j] = fmaxf(h2v[4 * r + 2 + j], 0.f);
          part0 = fmaf(h2v[4 * r + j], w, part0);
          part1 = fmaf(h2v[4 * r + 2 + j], w, part1);
        }
      part0 += __shfl_xor_sync(0xffffffffu, part0, 1);
      part0 += __shfl_xor_sync(0xffffffffu, part0, 2);
      part1 += __shfl_xor_sync(0xffffffffu, part1, 1);
      part1 += __shfl_xor_sync(0xffffffffu, part1, 2);
      if ((lane & 3) == 0) {
        sHead[wq * P + p0] = part0;
        sHead[wq * P + p1] = part1;
      }
    }
    // the four warps of this lane quarter (warps q, q+4, q+8, q+12) own rows 16q..16q+15: they
    // exchange their partial heads among themselves (named barrier 2 + q), no CTA barrier
    umma::named_sync(2 + quarter, 128);
    {
      float gg[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int pr = k ? p1 : p0;
        gg[k] = 0.f;
        if (pr < cnt) {
          float raw = sHead[pr];
#pragma unroll
          for (int q = 1; q < WQ; ++q) raw += sHead[q * P + pr];
          const float y = __fadd_rn(__fmul_rn(raw, md.span), md.vmin);
          const float r = __fsub_rn(y, cT[pr]);
          const float sqe = __fmul_rn(r, r);
          if (wq == 0 && (lane & 3) == 0) {  // one writer per point
            a.sq[tile * P + pr] = sqe;
            loss += double(sqe);
          }
          gg[k] = __fmul_rn(r, coef);
        }
      }
      const float g0 = gg[0], g1 = gg[1];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        float d0[2], d1[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const float w = sW3[ep_col0 + 8 * r + ec + j];
          const float a0 = h2v[4 * r + j], a1 = h2v[4 * r + 2 + j];
          dw3_acc[2 * r + j] = fmaf(g1, a1, fmaf(g0, a0, dw3_acc[2 * r + j]));
          d0[j] = a0 > 0.f ? __fmul_rn(g0, w) : 0.f;  // g_z2 (optim.py:143-145)
          d1[j] = a1 > 0.f ? __fmul_rn(g1, w) : 0.f;
        }
        umma::store_pair2(DZ2, PL64x64, p0, ep_col0 + 8 * r + ec, 64, d0[0], d0[1]);
        umma::store_pair2(DZ2, PL64x64, p1, ep_col0 + 8 * r + ec, 64, d1[0], d1[1]);
      }
    }
    umma::fence_async_smem();
    umma::fence_before_sync();
    // only the issuing warp waits for the stores; the others go on to their share of the
    // previous tile's scatter
    handoff(BAR_MMA);
    umma::fence_after_sync();
    TC16_STAMP(4);
    // ---- dz1 = dz2 W2 (-> acc A), dW2 += dz2^T h1 (-> TMEM sum) ----
    if constexpr (!kMmaWarp) issue_dz1_dw2();
    if (cnt_prev >= 0)
      scatter_pairs<FX>(md, a, GF, cache_prev, SQ2, SQ3, cnt_prev, warp, lane);
    TC16_WSTAMP(14);
    umma::mbar_wait(bar, phase);
    phase ^= 1;
    umma::fence_after_sync();
    TC16_STAMP(5);
    // ---- dz1 *= [h1 > 0] -> bf16x3 (same elements as this thread's epilogue 1) ----
    {
      float v[8];
      umma::tmem_ld_16x256b_x2(TA + lane_base + ep_col0, v);
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (!((h1pos >> e) & 1u)) v[e] = 0.f;
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        umma::store_pair2(DZ1, PL64x64, p0, ep_col0 + 8 * r + ec, 64, v[4 * r], v[4 * r + 1]);
        umma::store_pair2(DZ1, PL64x64, p1, ep_col0 + 8 * r + ec, 64, v[4 * r + 2], v[4 * r + 3]);
      }
    }
    umma::fence_async_smem();
    umma::fence_before_sync();
    // only the issuing warp waits for the stores; the others go on to their share of the
    // previous tile's scatter
    handoff(BAR_MMA);
    umma::fence_after_sync();
    TC16_STAMP(6);
    // ---- gF = dz1 W1 (-> acc A|B, N=128), dW1 += dz1^T F (-> TMEM sum) ----
    if constexpr (!kMmaWarp) issue_gf_dw1();
    if (cnt_prev >= 0) scatter_pairs<FX>(md, a, GF, cache_prev, SQ3, SQ, cnt_prev, warp, lane);
    TC16_WSTAMP(15);
    umma::mbar_wait(bar, phase);
    phase ^= 1;
    dw1_pending = kSplitDW1;  // this tile's dW1 completes on bar + 1
    umma::fence_after_sync();
    umma::fence_before_sync();
    worker_sync();  // every warp's scatter of the previous tile has read gF before it is overwritten
    umma::fence_after_sync();
    TC16_STAMP(7);
    // ---- gF epilogue: 32 columns per warp -> gF[p][k] ----
    {
      float v[16];
      umma::tmem_ld_16x256b_x4(TA + lane_base + 2 * ep_col0, v);
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int k = 2 * ep_col0 + 8 * r + ec;
        *reinterpret_cast<float2*>(GF + gf_idx(p0, k)) = make_float2(v[4 * r], v[4 * r + 1]);
        *reinterpret_cast<float2*>(GF + gf_idx(p1, k)) = make_float2(v[4 * r + 2], v[4 * r + 3]);
      }
    }
    umma::fence_before_sync();
    worker_sync();
    TC16_STAMP(8);
    // ---- encode of the next tile with the first SQ_I pairs of this tile's scatter interleaved;
    // the rest of the scatter runs in the next tile's tensor-core waits ----
    const int64_t next = tile + gridDim.x;
    if (next < tiles) {
      encode_tile(sX + ((it + 1) & 1) * 3 * P, cache_prev, cache_cur, cnt, next + gridDim.x, it + 2);
      cnt_prev = cnt;
    } else {
      scatter_pairs<FX>(md, a, GF, cache_cur, 0, SQ, cnt, warp, lane);
    }
  }

  // ---- flush per-CTA partials: [dW1 (64x128) | dW2 (64x64) | dW3 (64)] from TMEM ----
  if (dw1_pending) {  // the last tile's dW1
    umma::mbar_wait(bar + 1, phase_dw1);
    phase_dw1 ^= 1;
  }
  umma::fence_before_sync();
  worker_sync();
  umma::fence_after_sync();
  float* dst = a.part_dw + int64_t(blockIdx.x) * (HID * FE + HID * HID + HID);
  {
    float v[16];
    umma::tmem_ld_16x256b_x4(TDW1 + lane_base + 2 * ep_col0, v);  // dW1 rows i = p0 / p1
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int k = 2 * ep_col0 + 8 * r + ec;
      dst[p0 * FE + k] = v[4 * r];
      dst[p0 * FE + k + 1] = v[4 * r + 1];
      dst[p1 * FE + k] = v[4 * r + 2];
      dst[p1 * FE + k + 1] = v[4 * r + 3];
    }
    umma::tmem_ld_16x256b_x2(TDW2 + lane_base + ep_col0, v);  // dW2 rows j = p0 / p1
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int i = ep_col0 + 8 * r + ec;
      dst[HID * FE + p0 * HID + i] = v[4 * r];
      dst[HID * FE + p0 * HID + i + 1] = v[4 * r + 1];
      dst[HID * FE + p1 * HID + i] = v[4 * r + 2];
      dst[HID * FE + p1 * HID + i + 1] = v[4 * r + 3];
    }
  }
  // dW3: the 8 threads sharing lane & 3 hold the same columns
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    float v = dw3_acc[c];
    v += __shfl_xor_sync(0xffffffffu, v, 4);
    v += __shfl_xor_sync(0xffffffffu, v, 8);
    v += __shfl_xor_sync(0xffffffffu, v, 16);
    if (lane < 4) sDW3[quarter * HID + ep_col0 + 8 * (c >> 1) + ec + (c & 1)] = v;  // one writer per slot
  }
  // CTA sum over the worker warps (block_sum with the workers' barrier)
  auto worker_sum = [&](double v) {
    v = warp_sum(v);
    worker_sync();
    if (lane == 0) red[warp] = v;
    worker_sync();
    double t = (tid < NW) ? red[tid] : 0.0;
    if (warp == 0) t = warp_sum(t);
    if (tid == 0) red[0] = t;
    worker_sync();
    const double r = red[0];
    worker_sync();
    return r;
  };
  const double bl = worker_sum(loss);
  if (rho_on) {
    const double br = worker_sum(srho);
    if (tid == 0) {  // the rho pass's (sum rho, sum sq_err) partials, one pair per CTA
      md.rho_part[2 * blockIdx.x] = br;
      md.rho_part[2 * blockIdx.x + 1] = bl;
    }
  }
  if (tid < HID)  // fixed-order sum over the lane quarters: run-to-run deterministic
    dst[HID * FE + HID * HID + tid] = ((sDW3[tid] + sDW3[HID + tid]) + sDW3[2 * HID + tid]) + sDW3[3 * HID + tid];
  if (tid == 0) a.part_loss[blockIdx.x] = bl;
  umma::fence_before_sync();
  if constexpr (kMmaWarp) umma::named_sync(BAR_END, NT_LAUNCH); else __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tmem, TMEM_COLS);
}

}  // namespace tc16

extern "C" int apmg_debug_tc16_phases(long long* out) {
  APMG_CUDA_TRY(cudaMemcpyFromSymbol(out, tc16::g_tc16_stamp, sizeof(tc16::g_tc16_stamp)));
  return APMG_OK;
}
extern "C" int apmg_debug_tc16_warp_phases(long long* out) {  // [16 tiles][16 warps][16 points]
  APMG_CUDA_TRY(cudaMemcpyFromSymbol(out, tc16::g_tc16_wstamp, sizeof(tc16::g_tc16_wstamp)));
  return APMG_OK;
}

// the flagship shape (64 grids x 2 channels -> 128 features) runs this kernel; APMG_MLP=simt
// forces the SIMT tile kernel (A/B tests)
bool recon_tc_eligible(const ModelDev<float>& md) {
  const char* e = getenv("APMG_MLP");
  const bool tc_on = !(e && e[0] == 's');
  return tc_on && md.F == 128 && md.C == 2 && md.M == 64;
}

int launch_recon_tc16(const ModelDev<float>& md, int64_t n, const float* coords, const float* targets, float* sq,
                      float* dgrid, float* part_dw, double* part_loss, int grid, const TrainCtl* ctl,
                      cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    APMG_CUDA_TRY(cudaFuncSetAttribute(tc16::k_recon_tc16<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(tc16::SMEM_BYTES)));
    APMG_CUDA_TRY(cudaFuncSetAttribute(tc16::k_recon_tc16<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(tc16::SMEM_BYTES)));
    attr = true;
  }
  const char* ea = getenv("APMG_SCATTER_AGG");
  const char* es = getenv("APMG_TC_STAMPS");
  // APMG_SCATTER_AGG: 0 plain REDs, 1 tree-reduced, 2 (default) leader-gather aggregation
  tc16::Args a{md, n, coords, targets, sq, dgrid, part_dw, part_loss, ctl, ea ? atoi(ea) : 2,
               (es && es[0] == '1') ? 1 : 0};
  if (md.dgrid_fx) a.aggregate = 2;  // the fixed-point (deterministic) scatter lives in the gather variant
  if (md.dgrid_fx)
    APMG_LAUNCH("recon_fwd_bwd_tc", tc16::k_recon_tc16<true>, grid, tc16::NT_LAUNCH, tc16::SMEM_BYTES, st, a);
  else
    APMG_LAUNCH("recon_fwd_bwd_tc", tc16::k_recon_tc16<false>, grid, tc16::NT_LAUNCH, tc16::SMEM_BYTES, st, a);
  return APMG_OK;
}

}  // namespace apmg
