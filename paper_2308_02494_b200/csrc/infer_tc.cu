// Tensor-core lattice sweep (trainer.py:226-247 psnr, decomposition.py:294-304 brick boxes)
// for the flagship shape (float32, 64 grids x 2 channels -> 128 features, 64 hidden).
//
// One persistent CTA (16 warps) per SM, 64-voxel tiles, software-pipelined so that both
// tensor-core products hide behind CUDA-core work:
//     encode(t) | z1(t) issue | head(t-1) [z2(t-1) wait] | z1 wait, epilogue 1 -> h1 |
//     z2(t) issue | encode(t+1) ...
//   encode   lattice voxel -> f32 coordinate (the reference casts the f64 lattice
//            coordinate to float32 before predicting) -> per-grid f32 cell math -> features
//            split into TF32 hi/lo in the CM layout
//   z1, z2   tcgen05.mma kind::tf32, M=64, N=64, 3 products (3xTF32)
//   head     out = relu(z2) w3 * span + vmin; reconstruct-to-HBM and / or f64 SSE vs truth
// Features use f32 lerps (<= 1 ulp from the bit-exact f64-lerp encoder of k_forward);
// outputs agree with the reference forward to ~1e-6 relative (forward gate 1e-4).
#include "fwd_args.cuh"
#include "umma.cuh"

namespace apmg {
namespace itc {

constexpr int P = 64;
constexpr int NW = 16;
constexpr int NT = 32 * NW;
constexpr int WQ = NW / 4;
constexpr int EPC = 64 / WQ;
constexpr int GPW = 64 / NW;
constexpr int FE = 128;
constexpr int HID = 64;

// weights as stacked [hi rows; lo rows] CM buffers (R = 128): one N=128 product gives
// X.Whi and X.Wlo side by side, a second N=64 product adds Xlo.Whi onto the lo half
constexpr uint32_t OFF_W1S = 0;                        // [128][128]
constexpr uint32_t OFF_W2S = OFF_W1S + 128 * 128 * 4;  // [128][64]
constexpr uint32_t OFF_FH = OFF_W2S + 128 * 64 * 4;
constexpr uint32_t OFF_FL = OFF_FH + P * FE * 4;
constexpr uint32_t OFF_H1H = OFF_FL + P * FE * 4;
constexpr uint32_t OFF_H1L = OFF_H1H + P * HID * 4;
constexpr uint32_t OFF_X = OFF_H1L + P * HID * 4;     // [2][P][3] (tile parity)
constexpr uint32_t OFF_TRU = OFF_X + 2 * P * 3 * 4;   // [3][P] truth values (tile index mod 3)
constexpr uint32_t OFF_HEAD = OFF_TRU + 3 * P * 4;    // [WQ][P]
constexpr uint32_t OFF_RED = OFF_HEAD + WQ * P * 4;   // [32] doubles
constexpr uint32_t OFF_BAR = OFF_RED + 32 * 8;        // 2 mbarriers
constexpr uint32_t OFF_TM = OFF_BAR + 16;
constexpr uint32_t OFF_TF = OFF_TM + 16;              // [64][12]
constexpr uint32_t OFF_W3 = OFF_TF + 64 * 12 * 4;     // [64]
constexpr uint32_t SMEM_BYTES = OFF_W3 + 64 * 4;
static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
constexpr uint32_t TMEM_COLS = 256;  // z1 (hi | lo halves) | z2 (hi | lo halves)

// per-phase clock stamps of CTA 0 / thread 0 (APMG_INFER_STAMPS=1, tools/tc_phases.py --infer)
__device__ long long g_itc_stamp[16][8];
#define ITC_STAMP(k)                                                                 \
  do {                                                                               \
    if (a.stamps && blockIdx.x == 0 && tid == 0 && it < 16) g_itc_stamp[it][k] = clock64(); \
  } while (0)

__device__ __forceinline__ float* fptr(unsigned char* sm, uint32_t off) { return reinterpret_cast<float*>(sm + off); }
__device__ __forceinline__ uint32_t cm64(int r, int c) { return umma::cm_offset(r, c, 64) >> 2; }

// per-axis coordinate tables: the lattice coordinate of a voxel is separable (f64 lattice
// coordinate -> float32 -> optional f64 brick affine -> float32, fwd_point), so each axis
// is evaluated once per sweep instead of once per voxel (three f64 divisions)
__global__ void k_axis_tables(FwdArgs<float> a, float* __restrict__ tab) {
  const int n0 = a.bw, n1 = a.bh, n2 = int(ceil_div(a.n, int64_t(a.bw) * a.bh));
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n0 + n1 + n2; e += gridDim.x * blockDim.x) {
    int axis, k;
    if (e < n0) {
      axis = 0, k = e;
    } else if (e < n0 + n1) {
      axis = 1, k = e - n0;
    } else {
      axis = 2, k = e - n0 - n1;
    }
    const int L = axis == 0 ? a.LW : (axis == 1 ? a.LH : a.LD);
    const int b0 = axis == 0 ? a.bx0 : (axis == 1 ? a.by0 : a.bz0);
    double g = double(__double2float_rn(lattice_coord(b0 + k, L)));
    if (a.affine) {
      const double sc = axis == 0 ? a.sc0 : (axis == 1 ? a.sc1 : a.sc2);
      const double of = axis == 0 ? a.of0 : (axis == 1 ? a.of1 : a.of2);
      g = add_rn(mul_rn(g, sc), of);
    }
    tab[e] = __double2float_rn(g);
  }
}

// truth / recon element of point i of the box (x fastest)
__device__ __forceinline__ int64_t voxel_of(const FwdArgs<float>& a, int64_t i) {
  const int64_t plane = int64_t(a.bw) * a.bh;
  const int z = int(i / plane);
  const int64_t r = i - z * plane;
  const int y = int(r / a.bw);
  const int x = int(r - int64_t(y) * a.bw);
  return lattice_elem(a, x, y, z);
}

__global__ void __launch_bounds__(NT, 1) k_infer_tc(FwdArgs<float> a, const float* __restrict__ tab) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const ModelDev<float>& md = a.md;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int quarter = warp & 3, wq = warp >> 2;
  float* W1s = fptr(sm, OFF_W1S);
  float* W2s = fptr(sm, OFF_W2S);
  float* Fh = fptr(sm, OFF_FH);
  float* Fl = fptr(sm, OFF_FL);
  float* H1h = fptr(sm, OFF_H1H);
  float* H1l = fptr(sm, OFF_H1L);
  float* sX = fptr(sm, OFF_X);
  float* sHead = fptr(sm, OFF_HEAD);
  float* sTru = fptr(sm, OFF_TRU);
  double* red = reinterpret_cast<double*>(sm + OFF_RED);
  uint64_t* bar1 = reinterpret_cast<uint64_t*>(sm + OFF_BAR);
  uint64_t* bar2 = bar1 + 1;
  uint32_t* tm_slot = reinterpret_cast<uint32_t*>(sm + OFF_TM);
  float* sTF = fptr(sm, OFF_TF);
  float* sW3 = fptr(sm, OFF_W3);

  for (int e = tid; e < 64 * 128; e += NT) {
    float hi, lo;
    umma::split_tf32(md.w1[e], hi, lo);
    W1s[umma::cm_offset(e >> 7, e & 127, 128) >> 2] = hi;
    W1s[umma::cm_offset(64 + (e >> 7), e & 127, 128) >> 2] = lo;
  }
  for (int e = tid; e < 64 * 64; e += NT) {
    float hi, lo;
    umma::split_tf32(md.w2[e], hi, lo);
    W2s[umma::cm_offset(e >> 6, e & 63, 128) >> 2] = hi;
    W2s[umma::cm_offset(64 + (e >> 6), e & 63, 128) >> 2] = lo;
  }
  for (int e = tid; e < 64 * 12; e += NT) sTF[e] = md.tf[16 * (e / 12) + (e % 12)];
  if (tid < HID) sW3[tid] = md.w3[tid];
  if (warp == 0) umma::tmem_alloc(tm_slot, TMEM_COLS);
  if (tid == 0) {
    umma::mbar_init(bar1, 1);
    umma::mbar_init(bar2, 1);
    umma::fence_mbar_init();
  }
  umma::fence_async_smem();
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tmem = *tm_slot;
  const uint32_t TZ1 = tmem, TZ2 = tmem + 128;
  const uint32_t lane_base = uint32_t(32 * quarter) << 16;
  const uint32_t sW1s = umma::smem_u32(W1s), sW2s = umma::smem_u32(W2s), sFh = umma::smem_u32(Fh),
                 sFl = umma::smem_u32(Fl), sH1h = umma::smem_u32(H1h), sH1l = umma::smem_u32(H1l);
  const uint32_t idesc64 = umma::idesc_tf32(64, 64, false, false), idesc128 = umma::idesc_tf32(64, 128, false, false);
  const int ep_row = 16 * quarter + lane;
  const int ep_col0 = EPC * wq;
  uint32_t ph1 = 0, ph2 = 0;
  double sse = 0.0;

  // head of a finished tile: relu(z2) . w3 -> output / SSE (waits for its z2)
  auto head = [&](int64_t tile, int par) {
    umma::mbar_wait(bar2, ph2);
    ph2 ^= 1;
    umma::fence_after_sync();
    float v[EPC], w[EPC];
    umma::tmem_ld16(TZ2 + lane_base + ep_col0, v);
    umma::tmem_ld16(TZ2 + lane_base + 64 + ep_col0, w);
    if (lane < 16) {
      float part = 0.f;
#pragma unroll
      for (int c = 0; c < EPC; ++c) part = fmaf(fmaxf(v[c] + w[c], 0.f), sW3[ep_col0 + c], part);
      sHead[wq * P + ep_row] = part;
    }
    umma::fence_before_sync();
    __syncthreads();
    if (tid < P) {
      const int64_t i = tile * P + tid;
      if (i < a.n) {
        float raw = sHead[tid];
#pragma unroll
        for (int q = 1; q < WQ; ++q) raw += sHead[q * P + tid];
        const float y = __fadd_rn(__fmul_rn(raw, md.span), md.vmin);
        if (a.recon) a.recon[voxel_of(a, i)] = y;
        if (a.truth) {
          const double d = sub_rn(double(y), double(sTru[par * P + tid]));  // par: tile index mod 3
          sse += d * d;
        }
      }
    }
  };

  const int64_t tiles = ceil_div(a.n, P);
  const float* tx = tab;
  const float* ty = tab + a.bw;
  const float* tz = tab + a.bw + a.bh;
  int64_t prev = -1;
  int it = 0;
  // coordinates (axis-table lookups) and truth values of one tile into parity buffers
  auto load_coords = [&](int64_t tile, int slot) {
    const int t = tid - (NT - P);  // the last two warps (warp 0 issues the MMAs)
    if (t < 0) return;
    float x0 = 0.f, x1 = 0.f, x2 = 0.f, tv = 0.f;
    const int64_t i = tile * P + t;
    if (tile < tiles && i < a.n) {
      const int64_t plane = int64_t(a.bw) * a.bh;
      const int z = int(i / plane);
      const int64_t r = i - z * plane;
      const int y = int(r / a.bw), x = int(r - int64_t(y) * a.bw);
      x0 = tx[x];
      x1 = ty[y];
      x2 = tz[z];
      if (a.truth) tv = a.truth[lattice_elem(a, x, y, z)];
    }
    float* d = sX + (slot & 1) * 3 * P;
    d[3 * t] = x0;
    d[3 * t + 1] = x1;
    d[3 * t + 2] = x2;
    sTru[(slot % 3) * P + t] = tv;
  };
  load_coords(blockIdx.x, 0);
  __syncthreads();
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++it) {
    ITC_STAMP(0);
    const float* cX = sX + (it & 1) * 3 * P;
    // ---- encode (overlaps the z2 product of the previous tile) ----
    {
      const float xa[2][3] = {{cX[3 * lane], cX[3 * lane + 1], cX[3 * lane + 2]},
                              {cX[3 * (lane + 32)], cX[3 * (lane + 32) + 1], cX[3 * (lane + 32) + 2]}};
#pragma unroll 1
      for (int jq = 0; jq < GPW / 2; ++jq) {
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
          float f0 = 0.f, f1 = 0.f;
          if (inside)
            interp_pair_f32(md.grid, md.W, md.H * md.W, ((m * md.D + iz) * md.H + iy) * md.W + ix, float(fxd),
                            float(fyd), float(fzd), f0, f1);
          float hi0, lo0, hi1, lo1;
          umma::split_tf32(f0, hi0, lo0);
          umma::split_tf32(f1, hi1, lo1);
          const uint32_t o = cm64(p, 2 * m);
          *reinterpret_cast<float2*>(Fh + o) = make_float2(hi0, hi1);
          *reinterpret_cast<float2*>(Fl + o) = make_float2(lo0, lo1);
        }
      }
    }
    umma::fence_async_smem();
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    ITC_STAMP(2);
    if (tid == 0) {
      for (int kk = 0; kk < FE / 8; ++kk) {
        const uint64_t fh = umma::desc_kmajor(sFh, 64, kk), fl = umma::desc_kmajor(sFl, 64, kk);
        const uint64_t ws = umma::desc_kmajor(sW1s, 128, kk);
        umma::mma_tf32(TZ1, fh, ws, idesc128, kk > 0);  // [Fh.Whi | Fh.Wlo]
        umma::mma_tf32(TZ1 + 64, fl, ws, idesc64, 1);   // lo half += Flo.Whi
      }
      umma::commit(bar1);
    }
    load_coords(tile + gridDim.x, it + 1);  // next tile's inputs (slots not read until then)
    // ---- head of the previous tile (overlaps z1 of this one) ----
    if (prev >= 0) head(prev, (it + 2) % 3);
    ITC_STAMP(3);
    // ---- epilogue 1 ----
    umma::mbar_wait(bar1, ph1);
    ph1 ^= 1;
    umma::fence_after_sync();
    {
      float v[EPC], w[EPC];
      umma::tmem_ld16(TZ1 + lane_base + ep_col0, v);
      umma::tmem_ld16(TZ1 + lane_base + 64 + ep_col0, w);
      if (lane < 16) {
#pragma unroll
        for (int c4 = 0; c4 < EPC; c4 += 4) {
          float hi[4], lo[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) umma::split_tf32(fmaxf(v[c4 + e] + w[c4 + e], 0.f), hi[e], lo[e]);
          const uint32_t o = cm64(ep_row, ep_col0 + c4);
          *reinterpret_cast<float4*>(H1h + o) = make_float4(hi[0], hi[1], hi[2], hi[3]);
          *reinterpret_cast<float4*>(H1l + o) = make_float4(lo[0], lo[1], lo[2], lo[3]);
        }
      }
    }
    umma::fence_async_smem();
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    if (tid == 0) {
      for (int kk = 0; kk < HID / 8; ++kk) {
        const uint64_t hh = umma::desc_kmajor(sH1h, 64, kk), hl = umma::desc_kmajor(sH1l, 64, kk);
        const uint64_t ws = umma::desc_kmajor(sW2s, 128, kk);
        umma::mma_tf32(TZ2, hh, ws, idesc128, kk > 0);
        umma::mma_tf32(TZ2 + 64, hl, ws, idesc64, 1);
      }
      umma::commit(bar2);
    }
    ITC_STAMP(4);
    prev = tile;
  }
  if (prev >= 0) head(prev, (it + 2) % 3);
  if (a.truth) {
    const double s = block_sum(sse, red);
    if (tid == 0) atomicAdd(a.sse, s);
  }
  umma::fence_before_sync();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tmem, TMEM_COLS);
}

}  // namespace itc

extern "C" int apmg_debug_infer_phases(long long* out) {
  APMG_CUDA_TRY(cudaMemcpyFromSymbol(out, itc::g_itc_stamp, sizeof(itc::g_itc_stamp)));
  return APMG_OK;
}

bool infer_tc_eligible(const FwdArgs<float>& a) {
  const char* e = getenv("APMG_MLP");  // APMG_MLP=simt keeps the SIMT sweep (A/B tests)
  return !(e && e[0] == 's') && a.mode == kFwdLattice && a.md.F == 128 && a.md.C == 2 && a.md.M == 64;
}

int launch_infer_tc(const FwdArgs<float>& a, cudaStream_t st) {
  static float* tab = nullptr;  // per-axis coordinate tables (grown on demand, never freed)
  static int64_t tab_cap = 0;
  const int64_t need = int64_t(a.bw) + a.bh + ceil_div(a.n, int64_t(a.bw) * a.bh);
  if (need > tab_cap) {
    if (tab) APMG_CUDA_TRY(cudaFree(tab));
    APMG_CUDA_TRY(cudaMalloc(&tab, sizeof(float) * need));
    tab_cap = need;
  }
  APMG_LAUNCH("infer_axis_tables", itc::k_axis_tables, int(ceil_div(need, 256)), 256, 0, st, a, tab);
  static bool attr = false;
  if (!attr) {
    APMG_CUDA_TRY(cudaFuncSetAttribute(itc::k_infer_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(itc::SMEM_BYTES)));
    attr = true;
  }
  const int64_t tiles = ceil_div(a.n, itc::P);
  const int grid = int(min64(tiles, int64_t(num_sms())));
  const char* es = getenv("APMG_INFER_STAMPS");
  FwdArgs<float> b = a;
  b.stamps = es && es[0] == '1';
  APMG_LAUNCH("infer_lattice_tc", itc::k_infer_tc, grid, itc::NT, itc::SMEM_BYTES, st, b, tab);
  return APMG_OK;
}

}  // namespace apmg
