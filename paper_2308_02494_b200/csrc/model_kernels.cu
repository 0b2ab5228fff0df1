// Encoder, fused forward and fused reconstruction forward/backward kernels.
//
// Reference: model.py:141-166 (encode/decode/forward), optim.py:76-155
// (_forward_chain, recon_loss_and_grads), trainer.py:226-247 (psnr sweep).
#include "kernels.cuh"
#include "fwd_args.cuh"

namespace apmg {

// ------------------------------------------------------------------ encode
template <typename T>
__global__ void __launch_bounds__(256) k_encode(ModelDev<T> md, const T* __restrict__ pts, int64_t n,
                                                T* __restrict__ feats) {
  const int64_t pairs = n * md.M;
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < pairs; q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = q / md.M;
    const int m = int(q - i * md.M);
    const T* x = pts + 3 * i;
    encode_grid_point(md, m, x[0], x[1], x[2], feats + i * md.F + int64_t(m) * md.C, 1);
  }
}

// ------------------------------------------------------------------ forward (FwdArgs: fwd_args.cuh)
template <typename T>
__global__ void __launch_bounds__(kTileThreads) k_forward(FwdArgs<T> a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const ModelDev<T>& md = a.md;
  const int F = md.F, Fs = feat_stride(F);
  T* sX = reinterpret_cast<T*>(smem_raw);          // [64][3]
  T* sF = sX + 3 * kTileP;                         // [64][Fs]
  T* sH1 = sF + kTileP * Fs;                       // [64][65]
  T* sH2 = sH1 + kTileP * kHS;                     // [64][65]
  __shared__ double red[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t tiles = ceil_div(a.n, kTileP);
  double sse = 0.0;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int64_t p0 = tile * kTileP;
    const int cnt = int(min64(kTileP, a.n - p0));
    if (a.mode == kFwdFeats) {
      for (int e = tid; e < kTileP * F; e += kTileThreads) {
        const int p = e / F, k = e - p * F;
        sF[p * Fs + k] = p < cnt ? a.feats[(p0 + p) * F + k] : T(0);
      }
      __syncthreads();
    } else {
      if (tid < kTileP) {
        T x0 = 0, x1 = 0, x2 = 0;
        if (tid < cnt) fwd_point(a, p0 + tid, x0, x1, x2);
        sX[3 * tid] = x0;
        sX[3 * tid + 1] = x1;
        sX[3 * tid + 2] = x2;
      }
      __syncthreads();
      // (point, grid) pairs: lane -> point, warp -> grid (transform loads are warp-uniform)
      for (int m = warp; m < md.M; m += kTileThreads / 32) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int p = lane + 32 * h;
          encode_grid_point(md, m, sX[3 * p], sX[3 * p + 1], sX[3 * p + 2], sF + p * Fs + m * md.C, 1);
        }
      }
      __syncthreads();
    }
    tile_dense(sF, Fs, F, md.w1, sH1, kHS, true);
    __syncthreads();
    tile_dense(sH1, kHS, kHidden, md.w2, sH2, kHS, true);
    __syncthreads();
    if (tid < cnt) {
      const T y = tile_head(sH2, md.w3, tid, md.span, md.vmin);
      const int64_t i = p0 + tid;
      if (a.mode == kFwdPts || a.mode == kFwdFeats) {
        a.out[i] = y;
      } else if (a.mode == kFwdGather) {
        a.gout[a.index[i]] = float(y);
      } else {
        const int64_t plane = int64_t(a.bw) * a.bh;
        const int z = int(i / plane);
        const int64_t r = i - z * plane;
        const int yy = int(r / a.bw);
        const int x = int(r - int64_t(yy) * a.bw);
        const int64_t v = lattice_elem(a, x, yy, z);
        if (a.recon) a.recon[v] = float(y);
        if (a.truth) {
          const double d = sub_rn(double(y), double(a.truth[v]));
          sse += d * d;
        }
      }
    }
    __syncthreads();
  }
  if (a.mode == kFwdLattice && a.truth) {
    const double s = block_sum(sse, red);
    if (tid == 0) a.sse_part[blockIdx.x] = s;
  }
}

// *sse += sum of the per-CTA parts in index order (one warp: fixed shuffle tree)
__global__ void k_sse_finalize(const double* __restrict__ part, int n, double* __restrict__ sse) {
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += 32) s += part[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if (threadIdx.x == 0) *sse += s;
}

int launch_sse_finalize(const double* part, int n, double* sse, cudaStream_t st) {
  APMG_LAUNCH("sse_finalize", k_sse_finalize, 1, 32, 0, st, part, n, sse);
  return APMG_OK;
}

template <typename T>
size_t forward_smem(int F) {
  return sizeof(T) * (3 * kTileP + size_t(kTileP) * feat_stride(F) + 2 * size_t(kTileP) * kHS);
}

template <typename T>
int launch_forward(const FwdArgs<T>& a, cudaStream_t st) {
  if (a.n <= 0) return APMG_OK;
  if constexpr (sizeof(T) == 4) {
    if (infer_tc_eligible(a)) return launch_infer_tc(a, st);
  }
  const size_t smem = forward_smem<T>(a.md.F);
  APMG_CUDA_TRY(cudaFuncSetAttribute(k_forward<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  int occ = 0;
  APMG_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_forward<T>, kTileThreads, smem));
  APMG_ARG_CHECK(occ > 0, "forward tile does not fit in shared memory (F=%d)", a.md.F);
  const int64_t tiles = ceil_div(a.n, kTileP);
  const int grid = int(min64(tiles, int64_t(num_sms()) * occ));
  FwdArgs<T> b = a;
  const bool sse = a.mode == kFwdLattice && a.truth;
  StreamScratch sse_s;
  if (sse) {
    sse_s = StreamScratch(sizeof(double) * grid, st);
    b.sse_part = sse_s.as<double>();
    APMG_ARG_CHECK(b.sse_part != nullptr, "out of device memory for the SSE partials");
  }
  APMG_LAUNCH("forward", k_forward<T>, grid, kTileThreads, smem, st, b);
  if (sse) return launch_sse_finalize(b.sse_part, grid, a.sse, st);
  return APMG_OK;  // scratch released (stream-ordered) by the guard
}

// ------------------------------------------------------------------ recon fwd+bwd
template <typename T>
struct ReconArgs {
  ModelDev<T> md;
  int64_t n;
  const T* coords;       // [n][3]
  const T* targets;      // [n]
  T* sq;                 // [n] per-point squared error
  T* dgrid;              // [M][D][H][W][C] accumulated
  T* part_dw;            // [gridDim][64F + 4096 + 64]
  double* part_loss;     // [gridDim]
  const TrainCtl* ctl;   // optional: skip when ctl->skip
};

template <typename T, bool kDwSmem>
__global__ void __launch_bounds__(kTileThreads) k_recon(ReconArgs<T> a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  if (a.ctl && a.ctl->skip) return;
  const ModelDev<T>& md = a.md;
  const int F = md.F, Fs = feat_stride(F);
  const int DW = kHidden * F + kHidden * kHidden + kHidden;
  T* sX = reinterpret_cast<T*>(smem_raw);  // [64][3]
  T* sT = sX + 3 * kTileP;                 // [64] targets
  T* sG = sT + kTileP;                     // [64] d loss / d raw
  T* sF = sG + kTileP;                     // [64][Fs] features, then d features
  T* sH1 = sF + kTileP * Fs;               // [64][65] h1, then d z1
  T* sH2 = sH1 + kTileP * kHS;             // [64][65] h2, then d z2
  T* dW = kDwSmem ? (sH2 + kTileP * kHS) : (a.part_dw + int64_t(blockIdx.x) * DW);
  T* dW1 = dW;                             // [64][F]
  T* dW2 = dW1 + kHidden * F;              // [64][64]
  T* dW3 = dW2 + kHidden * kHidden;        // [64]
  __shared__ double red[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < DW; e += kTileThreads) dW[e] = T(0);
  // coef = np.asarray(2/n, dtype) * span (optim.py:121)
  const T coef = mul_rn(T(2.0 / double(a.n)), md.span);
  double loss = 0.0;
  const int64_t tiles = ceil_div(a.n, kTileP);
  __syncthreads();
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int64_t p0 = tile * kTileP;
    const int cnt = int(min64(kTileP, a.n - p0));
    if (tid < kTileP) {
      const bool ok = tid < cnt;
      const int64_t i = p0 + tid;
      sX[3 * tid] = ok ? a.coords[3 * i] : T(0);
      sX[3 * tid + 1] = ok ? a.coords[3 * i + 1] : T(0);
      sX[3 * tid + 2] = ok ? a.coords[3 * i + 2] : T(0);
      sT[tid] = ok ? a.targets[i] : T(0);
    }
    __syncthreads();
    for (int m = warp; m < md.M; m += kTileThreads / 32) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int p = lane + 32 * h;
        encode_grid_point(md, m, sX[3 * p], sX[3 * p + 1], sX[3 * p + 2], sF + p * Fs + m * md.C, 1);
      }
    }
    __syncthreads();
    tile_dense(sF, Fs, F, md.w1, sH1, kHS, true);
    __syncthreads();
    tile_dense(sH1, kHS, kHidden, md.w2, sH2, kHS, true);
    __syncthreads();
    if (tid < kTileP) {  // head, residual, loss (optim.py:116-121)
      T g = T(0);
      if (tid < cnt) {
        const T y = tile_head(sH2, md.w3, tid, md.span, md.vmin);
        const T r = sub_rn(y, sT[tid]);
        const T s = mul_rn(r, r);
        a.sq[p0 + tid] = s;
        loss += double(s);
        g = mul_rn(r, coef);
      }
      sG[tid] = g;
    }
    __syncthreads();
    if (tid < kHidden) {  // dW3 = g^T h2
      T acc = T(0);
      for (int p = 0; p < kTileP; ++p) acc = fma(sG[p], sH2[p * kHS + tid], acc);
      dW3[tid] += acc;
    }
    __syncthreads();
    for (int e = tid; e < kTileP * kHidden; e += kTileThreads) {  // d z2 = (g w3) * (z2 > 0)
      const int p = e >> 6, j = e & 63;
      const T h = sH2[p * kHS + j];
      sH2[p * kHS + j] = h > T(0) ? mul_rn(sG[p], ldg(md.w3 + j)) : T(0);
    }
    __syncthreads();
    {  // dW2 += dz2^T h1 : thread -> row j = tid/4, 16 columns
      const int j = tid >> 2, i0 = (tid & 3) * 16;
      T acc[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) acc[q] = T(0);
      for (int p = 0; p < kTileP; ++p) {
        const T gz = sH2[p * kHS + j];
#pragma unroll
        for (int q = 0; q < 16; ++q) acc[q] = fma(gz, sH1[p * kHS + i0 + q], acc[q]);
      }
#pragma unroll
      for (int q = 0; q < 16; ++q) dW2[j * kHidden + i0 + q] += acc[q];
    }
    __syncthreads();
    {  // d z1 = (dz2 W2) * (z1 > 0), written over h1
      T acc0[8], acc1[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc0[q] = acc1[q] = T(0);
      for (int j = 0; j < kHidden; ++j) {
        const T g0 = sH2[lane * kHS + j], g1 = sH2[(lane + 32) * kHS + j];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const T wv = ldg(md.w2 + j * kHidden + 8 * warp + q);
          acc0[q] = fma(g0, wv, acc0[q]);
          acc1[q] = fma(g1, wv, acc1[q]);
        }
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        T* h0 = sH1 + lane * kHS + 8 * warp + q;
        T* h1 = sH1 + (lane + 32) * kHS + 8 * warp + q;
        *h0 = *h0 > T(0) ? acc0[q] : T(0);
        *h1 = *h1 > T(0) ? acc1[q] : T(0);
      }
    }
    __syncthreads();
    {  // dW1 += dz1^T F in 4x4 register blocks
      const int kb = (F + 3) / 4, nblk = 16 * kb;
      for (int b = tid; b < nblk; b += kTileThreads) {
        const int i0 = (b / kb) * 4, k0 = (b % kb) * 4;
        T acc[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[u][v] = T(0);
        for (int p = 0; p < kTileP; ++p) {
          T gz[4], f[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) gz[u] = sH1[p * kHS + i0 + u];
#pragma unroll
          for (int v = 0; v < 4; ++v) f[v] = (k0 + v < F) ? sF[p * Fs + k0 + v] : T(0);
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[u][v] = fma(gz[u], f[v], acc[u][v]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v)
            if (k0 + v < F) dW1[(i0 + u) * F + k0 + v] += acc[u][v];
      }
    }
    __syncthreads();
    // d features = dz1 W1, written over the feature tile
    for (int kc = 8 * warp; kc < F; kc += 64) {
      T acc0[8], acc1[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc0[q] = acc1[q] = T(0);
      for (int i = 0; i < kHidden; ++i) {
        const T g0 = sH1[lane * kHS + i], g1 = sH1[(lane + 32) * kHS + i];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const T wv = (kc + q < F) ? ldg(md.w1 + int64_t(i) * F + kc + q) : T(0);
          acc0[q] = fma(g0, wv, acc0[q]);
          acc1[q] = fma(g1, wv, acc1[q]);
        }
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (kc + q < F) {
          sF[lane * Fs + kc + q] = acc0[q];
          sF[(lane + 32) * Fs + kc + q] = acc1[q];
        }
      }
    }
    __syncthreads();
    // scatter d features into the grids (optim.py:129-152)
    for (int m = warp; m < md.M; m += kTileThreads / 32) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int p = lane + 32 * h;
        if (p < cnt)
          scatter_grid_point(md, a.dgrid, m, sX[3 * p], sX[3 * p + 1], sX[3 * p + 2], sF + p * Fs + m * md.C, 1);
      }
    }
    __syncthreads();
  }
  const double bl = block_sum(loss, red);
  if (tid == 0) a.part_loss[blockIdx.x] = bl;
  if (kDwSmem) {
    T* dst = a.part_dw + int64_t(blockIdx.x) * DW;
    for (int e = tid; e < DW; e += kTileThreads) dst[e] = dW[e];
  }
}

// Deterministic reduction of the per-CTA partials: w grads and the f64 loss.
constexpr int kFinLanes = 8;

template <typename T>
__global__ void k_recon_finalize(int nblocks, int F, const T* __restrict__ part_dw,
                                 const double* __restrict__ part_loss, int64_t n, T* dw1, T* dw2, T* dw3,
                                 double* loss, TrainCtl* ctl, double* l_rec_log) {
  if (ctl && ctl->skip) return;
  const int DW = kHidden * F + kHidden * kHidden + kHidden;
  // kFinLanes lanes per weight element, each summing every kFinLanes-th CTA partial, then a
  // shuffle tree: the 148-deep dependent add chain per element was latency-bound
  // (launched with kFinLanes * DW threads rounded up to whole blocks: every lane reaches the shuffles)
  const int sub = threadIdx.x % kFinLanes;
  {
    const int e = (blockIdx.x * blockDim.x + threadIdx.x) / kFinLanes;
    T acc = T(0);
    if (e < DW)
      for (int b = sub; b < nblocks; b += kFinLanes) acc += part_dw[int64_t(b) * DW + e];
#pragma unroll
    for (int o = kFinLanes / 2; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o, kFinLanes);
    if (sub == 0 && e < DW) {
    if (e < kHidden * F)
      dw1[e] = acc;
    else if (e < kHidden * F + kHidden * kHidden)
      dw2[e - kHidden * F] = acc;
    else
      dw3[e - kHidden * F - kHidden * kHidden] = acc;
    }
  }
  if (blockIdx.x == 0) {
    __shared__ double red[32];
    double s = 0.0;
    for (int b = threadIdx.x; b < nblocks; b += blockDim.x) s += part_loss[b];
    s = block_sum(s, red);
    if (threadIdx.x == 0) {
      const double l = s / double(n);
      if (loss) *loss = l;
      if (ctl) {
        ctl->l_rec = l;
        l_rec_log[ctl->it] = l;
      }
    }
  }
}

template <typename T>
size_t recon_smem(int F, bool dw_smem) {
  size_t e = 5 * size_t(kTileP) + size_t(kTileP) * feat_stride(F) + 2 * size_t(kTileP) * kHS;
  if (dw_smem) e += size_t(kHidden) * F + kHidden * kHidden + kHidden;
  return e * sizeof(T);
}

template <typename T>
int recon_plan(int F, int64_t n, bool& dw_smem, int& grid, size_t& smem) {
  static int max_smem = -1;
  if (max_smem < 0) {
    int dev = 0;
    APMG_CUDA_TRY(cudaGetDevice(&dev));
    APMG_CUDA_TRY(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  }
  dw_smem = recon_smem<T>(F, true) <= size_t(max_smem);
  smem = recon_smem<T>(F, dw_smem);
  APMG_ARG_CHECK(smem <= size_t(max_smem), "recon tile does not fit in shared memory (F=%d)", F);
  int occ = 0;
  if (dw_smem) {
    APMG_CUDA_TRY(cudaFuncSetAttribute(k_recon<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    APMG_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_recon<T, true>, kTileThreads, smem));
  } else {
    APMG_CUDA_TRY(cudaFuncSetAttribute(k_recon<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    APMG_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_recon<T, false>, kTileThreads, smem));
  }
  APMG_ARG_CHECK(occ > 0, "recon kernel cannot be resident (F=%d)", F);
  grid = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, kTileP), int64_t(num_sms()) * occ)));
  return APMG_OK;
}

template <typename T>
size_t recon_ws_bytes(int F, int64_t n) {
  bool dws;
  int grid;
  size_t smem;
  if (recon_plan<T>(F, n, dws, grid, smem) != APMG_OK) grid = 4 * 148;
  const size_t DW = size_t(kHidden) * F + kHidden * kHidden + kHidden;
  Carver c(nullptr, 0);
  c.take<T>(size_t(grid) * DW);
  c.take<double>(grid);
  return c.used + 256;
}

int recon_tc16_grid(int64_t n) { return int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 64), num_sms()))); }

bool recon_uses_tc16(const apmg_model& m) {
  if (m.dtype != APMG_F32) return false;
  return recon_tc_eligible(make_model_dev<float>(m));
}

template <typename T>
int launch_recon(const ModelDev<T>& md, int64_t n, const T* coords, const T* targets, T* sq, double* loss,
                 T* dgrid, T* dw1, T* dw2, T* dw3, void* ws, size_t wsb, const TrainCtl* ctl, double* l_rec_log,
                 cudaStream_t st) {
  bool dws;
  int grid;
  size_t smem;
  int rc = recon_plan<T>(md.F, n, dws, grid, smem);
  if (rc) return rc;
  const size_t DW = size_t(kHidden) * md.F + kHidden * kHidden + kHidden;
  Carver c(ws, wsb);
  T* part_dw = c.take<T>(size_t(grid) * DW);
  double* part_loss = c.take<double>(grid);
  if (!c.ok()) {
    set_error("recon workspace too small: need %zu, have %zu", c.used, wsb);
    return APMG_E_WORKSPACE;
  }
  bool done = false;
  if constexpr (sizeof(T) == 4) {
    if (md.grad_pairs) APMG_ARG_CHECK(recon_tc_eligible(md), "x-pair gradients need the tc16 kernel");
    APMG_ARG_CHECK(!md.rho_out || recon_tc_eligible(md), "the fused density pass needs the tc16 kernel");
    if (recon_tc_eligible(md)) {  // flagship shape: the bf16x3 all-tcgen05 kernel
      grid = recon_tc16_grid(n);
      rc = launch_recon_tc16(md, n, coords, targets, sq, dgrid, part_dw, part_loss, grid, ctl, st);
      if (rc) return rc;
      done = true;
    }
  }
  if (!done) {
    ReconArgs<T> a{md, n, coords, targets, sq, dgrid, part_dw, part_loss, ctl};
    if (dws)
      APMG_LAUNCH("recon_fwd_bwd", (k_recon<T, true>), grid, kTileThreads, smem, st, a);
    else
      APMG_LAUNCH("recon_fwd_bwd", (k_recon<T, false>), grid, kTileThreads, smem, st, a);
  }
  const int fin_grid = int(ceil_div(int64_t(DW) * kFinLanes, 256));
  APMG_LAUNCH("recon_finalize", k_recon_finalize<T>, fin_grid, 256, 0, st, grid, md.F, part_dw, part_loss, n, dw1,
              dw2, dw3, loss, const_cast<TrainCtl*>(ctl), l_rec_log);
  return APMG_OK;
}

template int launch_recon<float>(const ModelDev<float>&, int64_t, const float*, const float*, float*, double*, float*,
                                 float*, float*, float*, void*, size_t, const TrainCtl*, double*, cudaStream_t);
template int launch_recon<double>(const ModelDev<double>&, int64_t, const double*, const double*, double*, double*,
                                  double*, double*, double*, double*, void*, size_t, const TrainCtl*, double*,
                                  cudaStream_t);
template size_t recon_ws_bytes<float>(int, int64_t);
template size_t recon_ws_bytes<double>(int, int64_t);

}  // namespace apmg

// ====================================================================== C ABI
using namespace apmg;

static int check_model(const apmg_model* m) {
  APMG_ARG_CHECK(m != nullptr, "null model");
  APMG_ARG_CHECK(m->dtype == APMG_F32 || m->dtype == APMG_F64, "dtype must be APMG_F32 or APMG_F64");
  APMG_ARG_CHECK(m->grids >= 1 && m->channels >= 1, "grids and channels must be >= 1");
  APMG_ARG_CHECK(m->depth >= 2 && m->height >= 2 && m->width >= 2, "grid resolution must be >= 2");
  APMG_ARG_CHECK(m->hidden == kHidden, "hidden width must be 64");
  APMG_ARG_CHECK(m->flat_top_p >= 1, "flat_top_p must be >= 1");
  return APMG_OK;
}

extern "C" int apmg_encode(const apmg_model* m, const void* pts, int64_t n, void* feats, void* stream) {
  int rc = check_model(m);
  if (rc) return rc;
  if (n <= 0) return APMG_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t pairs = n * m->grids;
  const int grid = int(std::min<int64_t>(ceil_div(pairs, 256), int64_t(num_sms()) * 16));
  if (m->dtype == APMG_F32)
    APMG_LAUNCH("encode", k_encode<float>, grid, 256, 0, st, make_model_dev<float>(*m), static_cast<const float*>(pts),
                n, static_cast<float*>(feats));
  else
    APMG_LAUNCH("encode", k_encode<double>, grid, 256, 0, st, make_model_dev<double>(*m),
                static_cast<const double*>(pts), n, static_cast<double*>(feats));
  return APMG_OK;
}

template <typename T>
static int fwd_common(const apmg_model* m, int mode, const void* src, int64_t n, void* out, void* stream) {
  FwdArgs<T> a{};
  a.md = make_model_dev<T>(*m);
  a.mode = mode;
  a.n = n;
  a.pts = static_cast<const T*>(src);
  a.feats = static_cast<const T*>(src);
  a.out = static_cast<T*>(out);
  return launch_forward<T>(a, static_cast<cudaStream_t>(stream));
}

extern "C" int apmg_decode(const apmg_model* m, const void* feats, int64_t n, void* out, void* stream) {
  int rc = check_model(m);
  if (rc) return rc;
  return m->dtype == APMG_F32 ? fwd_common<float>(m, kFwdFeats, feats, n, out, stream)
                              : fwd_common<double>(m, kFwdFeats, feats, n, out, stream);
}

extern "C" int apmg_forward(const apmg_model* m, const void* pts, int64_t n, void* out, void* stream) {
  int rc = check_model(m);
  if (rc) return rc;
  return m->dtype == APMG_F32 ? fwd_common<float>(m, kFwdPts, pts, n, out, stream)
                              : fwd_common<double>(m, kFwdPts, pts, n, out, stream);
}

extern "C" int apmg_forward_tc(const apmg_model* m, const float* pts, int64_t n, float* out, void* stream) {
  int rc = check_model(m);
  if (rc) return rc;
  APMG_ARG_CHECK(m->dtype == APMG_F32, "apmg_forward_tc needs a float32 model");
  FwdArgs<float> a{};
  a.md = make_model_dev<float>(*m);
  a.mode = kFwdPts;
  a.n = n;
  a.pts = pts;
  a.out = out;
  a.tc_points = 1;
  return launch_forward<float>(a, static_cast<cudaStream_t>(stream));
}

extern "C" size_t apmg_recon_workspace_bytes(const apmg_model* m, int64_t n) {
  if (!m) return 0;
  const int F = m->grids * m->channels;
  return m->dtype == APMG_F32 ? recon_ws_bytes<float>(F, n) : recon_ws_bytes<double>(F, n);
}

extern "C" int apmg_recon_loss_grads(const apmg_model* m, const void* coords, const void* targets, int64_t n,
                                     void* sq_errors, double* loss, void* const* grads, void* workspace,
                                     size_t workspace_bytes, void* stream) {
  int rc = check_model(m);
  if (rc) return rc;
  APMG_ARG_CHECK(n >= 1, "empty batch");
  APMG_ARG_CHECK(grads != nullptr, "null grads");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (m->dtype == APMG_F32)
    return launch_recon<float>(make_model_dev<float>(*m), n, static_cast<const float*>(coords),
                               static_cast<const float*>(targets), static_cast<float*>(sq_errors), loss,
                               static_cast<float*>(grads[0]), static_cast<float*>(grads[1]),
                               static_cast<float*>(grads[2]), static_cast<float*>(grads[3]), workspace,
                               workspace_bytes, nullptr, nullptr, st);
  return launch_recon<double>(make_model_dev<double>(*m), n, static_cast<const double*>(coords),
                              static_cast<const double*>(targets), static_cast<double*>(sq_errors), loss,
                              static_cast<double*>(grads[0]), static_cast<double*>(grads[1]),
                              static_cast<double*>(grads[2]), static_cast<double*>(grads[3]), workspace,
                              workspace_bytes, nullptr, nullptr, st);
}

template <typename T>
static int lattice_impl(const apmg_model* m, int32_t w, int32_t h, int32_t d, const int32_t* box, const double* sc,
                        const double* of, const float* truth, double* sse, float* recon, void* stream,
                        int box_local = 0) {
  FwdArgs<T> a{};
  a.box_local = box_local;
  a.md = make_model_dev<T>(*m);
  a.mode = kFwdLattice;
  a.LW = w;
  a.LH = h;
  a.LD = d;
  a.bx0 = box[0];
  a.by0 = box[2];
  a.bz0 = box[4];
  a.bw = box[1] - box[0] + 1;
  a.bh = box[3] - box[2] + 1;
  const int bd = box[5] - box[4] + 1;
  if (a.bw <= 0 || a.bh <= 0 || bd <= 0) return APMG_OK;
  a.n = int64_t(a.bw) * a.bh * bd;
  a.affine = sc != nullptr;
  if (sc) {
    a.sc0 = sc[0];
    a.sc1 = sc[1];
    a.sc2 = sc[2];
    a.of0 = of[0];
    a.of1 = of[1];
    a.of2 = of[2];
  }
  a.truth = truth;
  a.recon = recon;
  a.sse = sse;
  return launch_forward<T>(a, static_cast<cudaStream_t>(stream));
}

extern "C" int apmg_lattice_sweep(const apmg_model* m, int32_t w, int32_t h, int32_t d, const int32_t box[6],
                                  const double* scale, const double* offset, const float* truth, double* sse,
                                  float* recon, void* stream) {
  int rc = check_model(m);
  if (rc) return rc;
  APMG_ARG_CHECK(w >= 1 && h >= 1 && d >= 1, "lattice dims must be positive");
  APMG_ARG_CHECK(box[0] >= 0 && box[1] < w && box[2] >= 0 && box[3] < h && box[4] >= 0 && box[5] < d,
                 "lattice box out of range");
  APMG_ARG_CHECK(truth == nullptr || sse != nullptr, "truth given without sse accumulator");
  return m->dtype == APMG_F32 ? lattice_impl<float>(m, w, h, d, box, scale, offset, truth, sse, recon, stream)
                              : lattice_impl<double>(m, w, h, d, box, scale, offset, truth, sse, recon, stream);
}

extern "C" int apmg_brick_sweep(const apmg_model* m, int32_t w, int32_t h, int32_t d, const int32_t box[6],
                                const double* scale, const double* offset, const float* truth_box, double* sse,
                                float* recon_box, void* stream) {
  int rc = check_model(m);
  if (rc) return rc;
  APMG_ARG_CHECK(w >= 1 && h >= 1 && d >= 1, "lattice dims must be positive");
  APMG_ARG_CHECK(box[0] >= 0 && box[1] < w && box[2] >= 0 && box[3] < h && box[4] >= 0 && box[5] < d,
                 "lattice box out of range");
  APMG_ARG_CHECK(truth_box == nullptr || sse != nullptr, "truth given without sse accumulator");
  return m->dtype == APMG_F32
             ? lattice_impl<float>(m, w, h, d, box, scale, offset, truth_box, sse, recon_box, stream, 1)
             : lattice_impl<double>(m, w, h, d, box, scale, offset, truth_box, sse, recon_box, stream, 1);
}

// Grouped forward over one brick's point list (used by apmg_decomposed_forward).
int apmg_internal_forward_gather(const apmg_model* m, const double* sc, const double* of, const float* pts,
                                 const int32_t* index, int64_t n, float* out, cudaStream_t st, int tc) {
  int rc = check_model(m);
  if (rc) return rc;
  APMG_ARG_CHECK(m->dtype == APMG_F32, "decomposed inference supports float32 brick models");
  FwdArgs<float> a{};
  a.md = make_model_dev<float>(*m);
  a.mode = kFwdGather;
  a.n = n;
  a.affine = 1;
  a.sc0 = sc[0];
  a.sc1 = sc[1];
  a.sc2 = sc[2];
  a.of0 = of[0];
  a.of1 = of[1];
  a.of2 = of[2];
  a.gpts = pts;
  a.index = index;
  a.gout = out;
  a.tc_points = tc;  // tensor-core sweep kernel (renderer queries) instead of the exact forward
  return launch_forward<float>(a, st);
}

// to_local (model.py:179-182): local = pts . A^T + t for one 4x4 transform
namespace apmg {
template <typename T>
__global__ void k_to_local(const T* __restrict__ tf, const T* __restrict__ pts, int64_t n, T* __restrict__ out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const T x0 = pts[3 * i], x1 = pts[3 * i + 1], x2 = pts[3 * i + 2];
#pragma unroll
    for (int r = 0; r < 3; ++r) out[3 * i + r] = local_coord(x0, x1, x2, tf[4 * r], tf[4 * r + 1], tf[4 * r + 2], tf[4 * r + 3]);
  }
}
}  // namespace apmg

extern "C" int apmg_to_local(int32_t dtype, const void* transform, const void* pts, int64_t n, void* out,
                             void* stream) {
  if (n <= 0) return APMG_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), int64_t(num_sms()) * 8)));
  if (dtype == APMG_F32)
    APMG_LAUNCH("to_local", k_to_local<float>, grid, 256, 0, st, static_cast<const float*>(transform),
                static_cast<const float*>(pts), n, static_cast<float*>(out));
  else
    APMG_LAUNCH("to_local", k_to_local<double>, grid, 256, 0, st, static_cast<const double*>(transform),
                static_cast<const double*>(pts), n, static_cast<double*>(out));
  return APMG_OK;
}
