// Tensor-core lattice sweep (trainer.py:226-247 psnr, decomposition.py:294-304 brick boxes)
// for the flagship shape (float32, 64 grids x 2 channels -> 128 features, 64 hidden).
//
// One persistent CTA (16 warps) per SM, 128-voxel tiles (M=128 tcgen05 products: TMEM lane
// = voxel), software-pipelined so that both tensor-core products hide behind CUDA-core work:
//     encode(t) | z1(t) issue | head(t-1) [z2(t-1) wait] | z1 wait, epilogue 1 -> h1 |
//     z2(t) issue | encode(t+1) ...
//   encode   lattice voxel -> f32 coordinate (the reference casts the f64 lattice
//            coordinate to float32 before predicting) -> per-grid f32 cell math -> features
//   z1, z2   tcgen05.mma kind::f16 on bf16x3 operands (x = h + m + l, 8+8+8 significant bits;
//            6 products hh, hm, mh, hl, lh, mm: f32-level accuracy, each product exact in the
//            f32 accumulator)
//   head     out = relu(z2) w3 * span + vmin; reconstruct-to-HBM and / or f64 SSE vs truth
// Features use f32 lerps (<= 1 ulp from the bit-exact f64-lerp encoder of k_forward);
// outputs agree with the reference forward to ~1e-6 relative (forward gate 1e-4).
//
// Shared memory (221 KB): W1 (3 x 16 KB) | W2 (3 x 8 KB) | F [128][128] (3 x 32 KB) |
// h1 [128][64] (3 x 16 KB) | small.  Operands in the 16-bit CM layout of umma.cuh.
#include "fwd_args.cuh"
#include "umma.cuh"

namespace apmg {
namespace itc {

constexpr int P = 128;
constexpr int NW = 16;          // worker warps (encode, epilogues, head)
constexpr int NT = 32 * NW;     // worker threads (named barrier 1)
constexpr int NTA = NT + 32;    // + one warp that only issues the tensor-core products
constexpr int WQ = NW / 4;     // warps per TMEM lane quarter
constexpr int EPC = 64 / WQ;   // accumulator columns per warp in the epilogues (16)
constexpr int FE = 128;
constexpr int HID = 64;

constexpr uint32_t W1_PLANE = 64 * 128 * 2, W2_PLANE = 64 * 64 * 2, F_PLANE = P * FE * 2, H1_PLANE = P * HID * 2;
constexpr uint32_t OFF_W1 = 0;
constexpr uint32_t OFF_W2 = OFF_W1 + 3 * W1_PLANE;
constexpr uint32_t OFF_F = OFF_W2 + 3 * W2_PLANE;
constexpr uint32_t OFF_H1 = OFF_F + 3 * F_PLANE;
constexpr uint32_t OFF_X = OFF_H1 + 3 * H1_PLANE;     // [2][P][3] (tile parity)
constexpr uint32_t OFF_TRU = OFF_X + 2 * P * 3 * 4;   // [3][P] truth values (tile index mod 3)
constexpr uint32_t OFF_HEAD = OFF_TRU + 3 * P * 4;    // [WQ][P]
constexpr uint32_t OFF_RED = OFF_HEAD + WQ * P * 4;   // [32] doubles
#ifndef ITC_NQ
#define ITC_NQ 4
#endif
constexpr int NQ = ITC_NQ;  // z1 is issued in NQ K-slices, each as soon as its NW / NQ encoding warps are done
constexpr uint32_t OFF_BAR = OFF_RED + 32 * 8;        // mbarriers: z1 done, z2 done, h1 ready, F slice 0..NQ-1 ready
constexpr uint32_t OFF_TM = OFF_BAR + 8 * (3 + NQ);
constexpr uint32_t OFF_W3 = OFF_TM + 16;              // [64]
constexpr uint32_t OFF_TF = OFF_W3 + 64 * 4;          // [64][12] transforms (f32)
constexpr uint32_t SMEM_BYTES = OFF_TF + 64 * 12 * 4;
static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
constexpr uint32_t TMEM_COLS = 128;  // z1 | z2

// bf16x3 products q = 0..5: (A plane, B plane) = hh, hm, mh, hl, lh, mm (largest first)
__host__ __device__ constexpr int kPA(int q) { return q == 2 ? 1 : (q == 4 ? 2 : (q == 5 ? 1 : 0)); }
__host__ __device__ constexpr int kPB(int q) { return q == 1 ? 1 : (q == 3 ? 2 : (q == 5 ? 1 : 0)); }

// per-phase clock stamps of CTA 0 / thread 0 (APMG_INFER_STAMPS=1, tools/infer_phases.py)
__device__ long long g_itc_stamp[16][8];
#define ITC_STAMP(k)                                                                 \
  do {                                                                               \
    if (a.stamps && blockIdx.x == 0 && tid == 0 && it < 16) g_itc_stamp[it][k] = clock64(); \
  } while (0)

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

__global__ void __launch_bounds__(NTA, 1) k_infer_tc(FwdArgs<float> a, const float* __restrict__ tab) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const ModelDev<float>& md = a.md;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int quarter = warp & 3, wq = warp >> 2;
  unsigned char* W1 = sm + OFF_W1;
  unsigned char* W2 = sm + OFF_W2;
  unsigned char* F = sm + OFF_F;
  unsigned char* H1 = sm + OFF_H1;
  float* sX = reinterpret_cast<float*>(sm + OFF_X);
  float* sTru = reinterpret_cast<float*>(sm + OFF_TRU);
  float* sHead = reinterpret_cast<float*>(sm + OFF_HEAD);
  double* red = reinterpret_cast<double*>(sm + OFF_RED);
  uint64_t* bar1 = reinterpret_cast<uint64_t*>(sm + OFF_BAR);  // z1 committed
  uint64_t* bar2 = bar1 + 1;                                     // z2 committed
  uint64_t* barF = bar1 + 3;  // barF[s]: F columns of K-slice s written by worker warps s NW/NQ .. (s+1) NW/NQ - 1
  uint64_t* barH = bar1 + 2;                                     // h1 written by all worker warps
  uint32_t* tm_slot = reinterpret_cast<uint32_t*>(sm + OFF_TM);
  float* sW3 = reinterpret_cast<float*>(sm + OFF_W3);

  // weights: rows = output unit, 8-column chunks
  for (int e = tid; e < 64 * 16; e += NTA) {
    const int r = e >> 4, c0 = (e & 15) * 8;
    umma::store_chunk3(W1, W1_PLANE, r, c0, 64, md.w1 + r * FE + c0);
  }
  for (int e = tid; e < 64 * 8; e += NTA) {
    const int r = e >> 3, c0 = (e & 7) * 8;
    umma::store_chunk3(W2, W2_PLANE, r, c0, 64, md.w2 + r * HID + c0);
  }
  if (tid < HID) sW3[tid] = md.w3[tid];
  float* sTF = reinterpret_cast<float*>(sm + OFF_TF);
  for (int e = tid; e < 64 * 12; e += NTA) sTF[e] = md.tf[16 * (e / 12) + (e % 12)];
  if (warp == 0) umma::tmem_alloc(tm_slot, TMEM_COLS);
  if (tid == 0) {
    umma::mbar_init(bar1, 1);
    umma::mbar_init(bar2, 1);
    for (int q = 0; q < NQ; ++q) umma::mbar_init(barF + q, NW / NQ);
    umma::mbar_init(barH, NW);
    umma::fence_mbar_init();
  }
  umma::fence_async_smem();
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tmem = *tm_slot;
  const uint32_t TZ1 = tmem, TZ2 = tmem + 64;
  const uint32_t lane_base = uint32_t(32 * quarter) << 16;
  const uint32_t base16 = umma::smem_u32(sm) >> 4;  // descriptors: base16 + compile-time fields
  const uint32_t idesc = umma::idesc_bf16(128, 64, false, false);
  const int ep_row = 32 * quarter + lane;  // M=128 accumulator: row = lane
  const int ep_col0 = EPC * wq;
  uint32_t ph1 = 0, ph2 = 0;
  double sse = 0.0;
  int it = 0;

  // head of a finished tile: relu(z2) . w3 -> output / SSE (waits for its z2)
  auto head = [&](int64_t tile, int par) {
    umma::mbar_wait(bar2, ph2);
    ph2 ^= 1;
    umma::fence_after_sync();
    float v[EPC];
    umma::tmem_ld16(TZ2 + lane_base + ep_col0, v);
    float part = 0.f;
#pragma unroll
    for (int c = 0; c < EPC; ++c) part = fmaf(fmaxf(v[c], 0.f), sW3[ep_col0 + c], part);
    sHead[wq * P + ep_row] = part;
    umma::fence_before_sync();
    umma::named_sync(1, NT);  // worker warps only
    if (tid < P) {
      const int64_t i = tile * P + tid;
      if (i < a.n) {
        float raw = sHead[tid];
#pragma unroll
        for (int q = 1; q < WQ; ++q) raw += sHead[q * P + tid];
        const float y = __fadd_rn(__fmul_rn(raw, md.span), md.vmin);
        if (a.mode == kFwdPts) {
          a.out[i] = y;
        } else if (a.mode == kFwdGather) {
          a.gout[a.index[i]] = y;
        } else if (a.recon) {
          a.recon[voxel_of(a, i)] = y;
        }
        if (a.truth) {
          const double d = sub_rn(double(y), double(sTru[par * P + tid]));  // par: tile index mod 3
          sse += d * d;
        }
      }
    }
  };

  const int64_t tiles = ceil_div(a.n, P);
  if (warp == NW) {
    // ---- MMA warp: z1 when the workers' F is complete, z2 when their h1 is ----
    uint32_t pf = 0, ph = 0;
    for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
      // z1 in NQ K-slices: slice s as soon as warps s NW/NQ .. have encoded its grids, so all but
      // the last slice of the products overlap the slower warps' encode
#pragma unroll
      for (int sl = 0; sl < NQ; ++sl) {
        umma::mbar_wait(barF + sl, pf);
        umma::fence_after_sync();
        if (lane == 0) {
#pragma unroll
          for (int kk = sl * (FE / 16 / NQ); kk < (sl + 1) * (FE / 16 / NQ); ++kk)
#pragma unroll
            for (int q = 0; q < 6; ++q)
              umma::mma_bf16_c(TZ1, base16, umma::kmajor_c(OFF_F + kPA(q) * F_PLANE, P, kk),
                               umma::kmajor_c(OFF_W1 + kPB(q) * W1_PLANE, 64, kk), idesc, (kk | q) ? 1u : 0u);
        }
        __syncwarp();
      }
      pf ^= 1;
      if (lane == 0) {
        umma::commit(bar1);
      }
      __syncwarp();
      umma::mbar_wait(barH, ph);
      ph ^= 1;
      umma::fence_after_sync();
      if (lane == 0) {
#pragma unroll
        for (int kk = 0; kk < HID / 16; ++kk)
#pragma unroll
          for (int q = 0; q < 6; ++q)
            umma::mma_bf16_c(TZ2, base16, umma::kmajor_c(OFF_H1 + kPA(q) * H1_PLANE, P, kk),
                             umma::kmajor_c(OFF_W2 + kPB(q) * W2_PLANE, 64, kk), idesc, (kk | q) ? 1u : 0u);
        umma::commit(bar2);
      }
      __syncwarp();
    }
  } else {
    const float* tx = tab;
    const float* ty = tab + a.bw;
    const float* tz = tab + a.bw + a.bh;
    // coordinates (axis-table lookups) and truth values of one tile into parity buffers,
    // by the last four worker warps
    // split in two: fetch (global loads into registers, issued at the top of an iteration so
    // their latency hides behind the encode) and publish (smem stores after the encode)
    struct Pre {
      float x0, x1, x2, tv;
    };
    auto fetch_coords = [&](int64_t tile) {
      Pre r{0.f, 0.f, 0.f, 0.f};
      const int t = tid - (NT - P);
      const int64_t i = tile * P + t;
      if (a.mode != kFwdLattice) {  // point list / brick gather (renderer queries): fwd_point
        if (t >= 0 && tile < tiles && i < a.n) fwd_point(a, i, r.x0, r.x1, r.x2);
        return r;
      }
      if (t >= 0 && tile < tiles && i < a.n) {
        const int64_t plane = int64_t(a.bw) * a.bh;
        const int z = int(i / plane);
        const int64_t rr = i - z * plane;
        const int y = int(rr / a.bw), x = int(rr - int64_t(y) * a.bw);
        r.x0 = tx[x];
        r.x1 = ty[y];
        r.x2 = tz[z];
        if (a.truth) r.tv = a.truth[lattice_elem(a, x, y, z)];
      }
      return r;
    };
    auto publish_coords = [&](const Pre& r, int slot) {
      const int t = tid - (NT - P);
      if (t < 0) return;
      float* d = sX + (slot & 1) * 3 * P;
      d[3 * t] = r.x0;
      d[3 * t + 1] = r.x1;
      d[3 * t + 2] = r.x2;
      sTru[(slot % 3) * P + t] = r.tv;
    };
    auto load_coords = [&](int64_t tile, int slot) { publish_coords(fetch_coords(tile), slot); };
    load_coords(blockIdx.x, 0);
    umma::named_sync(1, NT);
    int64_t prev = -1;
    for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++it) {
      ITC_STAMP(0);
      const float* cX = sX + (it & 1) * 3 * P;
      const Pre nxt = fetch_coords(tile + gridDim.x);  // next tile's inputs, in flight during the encode
      // ---- encode (overlaps z2 of the previous tile): warp w owns grids 4w..4w+3, i.e.
      // feature columns 8w..8w+7 (one 16-B chunk per plane); lane -> points lane + 32h ----
      {
        const float* tfw = sTF + 12 * (4 * warp);
  #pragma unroll
        for (int hp = 0; hp < P / 64; ++hp) {  // two points per pass: lane + 64 hp, lane + 64 hp + 32
          const int pa = lane + 64 * hp, pb = pa + 32;
          const float2 X0 = make_float2(cX[3 * pa], cX[3 * pb]), X1 = make_float2(cX[3 * pa + 1], cX[3 * pb + 1]),
                       X2 = make_float2(cX[3 * pa + 2], cX[3 * pb + 2]);
          float fv[2][8];
  #pragma unroll
          for (int g = 0; g < 4; ++g) {
            const int m = 4 * warp + g;
            const float* tf = tfw + 12 * g;
            const float2 l0 = local_coord2(X0, X1, X2, tf[0], tf[1], tf[2], tf[3]);
            const float2 l1 = local_coord2(X0, X1, X2, tf[4], tf[5], tf[6], tf[7]);
            const float2 l2 = local_coord2(X0, X1, X2, tf[8], tf[9], tf[10], tf[11]);
            int ix[2], iy[2], iz[2];
            float fx[2], fy[2], fz[2];
            axis_term2(l0, md.W, ix[0], ix[1], fx[0], fx[1]);
            axis_term2(l1, md.H, iy[0], iy[1], fy[0], fy[1]);
            axis_term2(l2, md.D, iz[0], iz[1], fz[0], fz[1]);
            const float la[2][3] = {{l0.x, l1.x, l2.x}, {l0.y, l1.y, l2.y}};
            bool ins[2];
            int vb[2];
  #pragma unroll
            for (int k = 0; k < 2; ++k) {
              ins[k] = (fabsf(la[k][0]) <= 1.f) && (fabsf(la[k][1]) <= 1.f) && (fabsf(la[k][2]) <= 1.f);
              // straight-line: an outside pair gathers cell 0 and is zeroed afterwards
              vb[k] = ins[k] ? ((m * md.D + iz[k]) * md.H + iy[k]) * md.W + ix[k] : 0;
            }
            // both points' corner loads issued before the first lerp
            float f0[2], f1[2];
            if (md.gridq) {
              float b[2][16];
  #pragma unroll
              for (int k = 0; k < 2; ++k) gather_pairq_f32(md.gridq, md.H * md.W, vb[k], b[k]);
  #pragma unroll
              for (int k = 0; k < 2; ++k) lerp_pairq_f32(b[k], fx[k], fy[k], fz[k], f0[k], f1[k]);
            } else if (md.gridx) {
              float4 b[2][4];
  #pragma unroll
              for (int k = 0; k < 2; ++k) gather_pairx_f32(md.gridx, md.W, md.H * md.W, vb[k], b[k]);
  #pragma unroll
              for (int k = 0; k < 2; ++k) lerp_pairx_f32(b[k], fx[k], fy[k], fz[k], f0[k], f1[k]);
            } else {
              float2 b[2][8];
  #pragma unroll
              for (int k = 0; k < 2; ++k) gather_pair_f32(md.grid, md.W, md.H * md.W, vb[k], b[k]);
  #pragma unroll
              for (int k = 0; k < 2; ++k) lerp_pair_f32(b[k], fx[k], fy[k], fz[k], f0[k], f1[k]);
            }
  #pragma unroll
            for (int k = 0; k < 2; ++k) {
              fv[k][2 * g] = ins[k] ? f0[k] : 0.f;
              fv[k][2 * g + 1] = ins[k] ? f1[k] : 0.f;
            }
          }
          umma::store_chunk3(F, F_PLANE, pa, 8 * warp, P, fv[0]);
          umma::store_chunk3(F, F_PLANE, pb, 8 * warp, P, fv[1]);
        }
      }
      umma::fence_async_smem();
      __syncwarp();
      if (lane == 0) umma::mbar_arrive(barF + warp / (NW / NQ));  // this warp's F columns are in place
      ITC_STAMP(2);
      publish_coords(nxt, it + 1);  // next tile's inputs (slots not read until then)
      // ---- head of the previous tile (overlaps z1 of this one); its worker barrier also
      // publishes the coordinates just loaded (first tile: an explicit barrier) ----
      if (prev >= 0)
        head(prev, (it + 2) % 3);
      else
        umma::named_sync(1, NT);
      ITC_STAMP(3);
      // ---- epilogue 1: h1 = relu(z1) -> bf16x3 h1 rows ----
      umma::mbar_wait(bar1, ph1);
      ph1 ^= 1;
      umma::fence_after_sync();
      {
        float v[EPC];
        umma::tmem_ld16(TZ1 + lane_base + ep_col0, v);
  #pragma unroll
        for (int c = 0; c < EPC; ++c) v[c] = fmaxf(v[c], 0.f);
        umma::store_chunk3(H1, H1_PLANE, ep_row, ep_col0, P, v);
        umma::store_chunk3(H1, H1_PLANE, ep_row, ep_col0 + 8, P, v + 8);
      }
      umma::fence_async_smem();
      umma::fence_before_sync();
      __syncwarp();
      if (lane == 0) umma::mbar_arrive(barH);  // this warp's h1 rows are in place
      ITC_STAMP(4);
      prev = tile;
    }
    if (prev >= 0) head(prev, (it + 2) % 3);
  }
  if (a.truth) {
    const double s = block_sum(sse, red);
    if (tid == 0) a.sse_part[blockIdx.x] = s;
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
  return !(e && e[0] == 's') && (a.mode == kFwdLattice || ((a.mode == kFwdPts || a.mode == kFwdGather) && a.tc_points)) &&
         a.md.F == 128 && a.md.C == 2 && a.md.M == 64;
}

int launch_infer_tc(const FwdArgs<float>& a, cudaStream_t st) {
  // per-call scratch, stream-ordered: per-axis coordinate tables (lattice sweeps), the grid copy
  // (xy-quad, or x-pair), the per-CTA SSE partials
  StreamScratch tab_s, gx_s, sse_s;
  float* tab = nullptr;
  if (a.mode == kFwdLattice) {
    const int64_t need = int64_t(a.bw) + a.bh + ceil_div(a.n, int64_t(a.bw) * a.bh);
    tab_s = StreamScratch(sizeof(float) * need, st);
    tab = tab_s.as<float>();
    APMG_ARG_CHECK(tab != nullptr, "out of device memory for the sweep tables");
    APMG_LAUNCH("infer_axis_tables", itc::k_axis_tables, int(ceil_div(need, 256)), 256, 0, st, a, tab);
  }
  const int64_t cells = int64_t(a.md.M) * a.md.D * a.md.H * a.md.W;
  const char* eg = getenv("APMG_GRIDX");
  const char* eq = getenv("APMG_INFER_GRIDQ");
  // the xy-quad copy (ModelDev::gridq): 2 256-bit corner loads per (point, grid); measured against
  // the grid itself (lattice sweeps, 8 float2 loads: 2.57 vs 2.37 G voxels/s over 1024^3) and the
  // x-pair copy (point lists, 4 float4 loads: 512^2 x 128 render 18.0 vs 19.6 ms).
  // APMG_INFER_GRIDQ=0: those layouts (APMG_GRIDX=0: the grid itself for point lists too)
  const bool use_gq = !(eq && eq[0] == '0');
  const bool use_gx = !use_gq && a.mode != kFwdLattice && !(eg && eg[0] == '0');
  float4* gx = nullptr;
  if (use_gx || use_gq) {
    gx_s = StreamScratch(sizeof(float4) * (use_gq ? 2 * cells : cells), st);
    gx = gx_s.as<float4>();
    APMG_ARG_CHECK(gx != nullptr, "out of device memory for the grid copy");
    if (use_gq)
      APMG_LAUNCH("pack_gridq", k_pack_gridq, elementwise_grid(cells, 8), 256, 0, st,
                  reinterpret_cast<const float2*>(a.md.grid), gx, cells, a.md.W);
    else
      APMG_LAUNCH("pack_gridx", k_pack_gridx, elementwise_grid(cells, 8), 256, 0, st,
                  reinterpret_cast<const float2*>(a.md.grid), gx, cells);
  }
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
  b.md.gridx = use_gq ? nullptr : gx;
  b.md.gridq = use_gq ? reinterpret_cast<const float*>(gx) : nullptr;
  const bool sse = a.mode == kFwdLattice && a.truth;
  if (sse) {
    sse_s = StreamScratch(sizeof(double) * grid, st);
    b.sse_part = sse_s.as<double>();
    APMG_ARG_CHECK(b.sse_part != nullptr, "out of device memory for the SSE partials");
  }
  if (a.mode != kFwdLattice)
    APMG_LAUNCH("infer_points_tc", itc::k_infer_tc, grid, itc::NTA, itc::SMEM_BYTES, st, b, tab);
  else
    APMG_LAUNCH("infer_lattice_tc", itc::k_infer_tc, grid, itc::NTA, itc::SMEM_BYTES, st, b, tab);
  if (sse) return launch_sse_finalize(b.sse_part, grid, a.sse, st);
  return APMG_OK;  // scratch released (stream-ordered) by the guards
}

}  // namespace apmg
