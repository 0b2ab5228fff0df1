// Flat-top feature density, error-warped target, KL loss and the transform
// gradient, all in float64 (density.py:83-148, optim.py:158-200).
//
// Three passes over the batch with two tiny deterministic reductions between
// them (the loss needs sum(rho) before rho_scaled exists and sum(d_s * rho_s)
// before d_rho exists):
//   P1  per point: rho = sum_m |det_m| bump_m            -> rho[n], partial sums
//   P2  per point: rho_s, rho*, loss term, d_s            -> d_s[n], partial sums
//   P3  per (grid, chunk): 13 gradient accumulators      -> partials[chunk][m][13]
//   P4  per grid: dA = sign(det) W cof - 2p G, dt = -2p T (+ masked Adam in training)
#include "kernels.cuh"

namespace apmg {

constexpr double kEps = 1e-8;        // density.py:34
constexpr double kClamp = 700.0;     // density.py:35
constexpr double kFloor = 1e-300;    // density.py:39
constexpr int kDensThreads = 256;
constexpr int kMaxGridsSmem = 1024;  // transforms staged in smem (13 doubles each)

// x^(2p) computed from s = x*x as s^p by squaring (numpy uses its own pow; ULP-level differences)
__device__ __forceinline__ double powi(double s, int p) {
  double r = 1.0, b = s;
  bool first = true;
  while (p) {
    if (p & 1) {
      r = first ? b : r * b;
      first = false;
    }
    p >>= 1;
    if (p) b = b * b;
  }
  return first ? 1.0 : r;
}

// Stage f64 transforms (12 values) and det per grid in shared memory.
// det = a0 . (a1 x a2) with numpy's (t0 + t2) + t1 einsum order (density.py:98).
template <typename T>
__device__ void stage_transforms(const T* __restrict__ tf, int M, double* s_tf) {
  for (int m = threadIdx.x; m < M; m += blockDim.x) {
    double a[12];
#pragma unroll
    for (int e = 0; e < 12; ++e) a[e] = double(tf[16 * m + e]);
#pragma unroll
    for (int e = 0; e < 12; ++e) s_tf[13 * m + e] = a[e];
    const double c0 = sub_rn(mul_rn(a[5], a[10]), mul_rn(a[6], a[9]));
    const double c1 = sub_rn(mul_rn(a[6], a[8]), mul_rn(a[4], a[10]));
    const double c2 = sub_rn(mul_rn(a[4], a[9]), mul_rn(a[5], a[8]));
    s_tf[13 * m + 12] = add_rn(add_rn(mul_rn(a[0], c0), mul_rn(a[2], c2)), mul_rn(a[1], c1));
  }
}

// local coords of point x in grid with staged row-major A|t (density.py:97, (t0+t2)+t1 order)
__device__ __forceinline__ void dens_local(const double* a, double x0, double x1, double x2, double& l0, double& l1,
                                           double& l2) {
  l0 = add_rn(add_rn(add_rn(mul_rn(a[0], x0), mul_rn(a[2], x2)), mul_rn(a[1], x1)), a[3]);
  l1 = add_rn(add_rn(add_rn(mul_rn(a[4], x0), mul_rn(a[6], x2)), mul_rn(a[5], x1)), a[7]);
  l2 = add_rn(add_rn(add_rn(mul_rn(a[8], x0), mul_rn(a[10], x2)), mul_rn(a[9], x1)), a[11]);
}

__device__ __forceinline__ double bump_of(double l0, double l1, double l2, int p) {
  const double q = add_rn(add_rn(powi(l0 * l0, p), powi(l1 * l1, p)), powi(l2 * l2, p));
  return (q > kClamp || q != q) ? (q != q ? q : 0.0) : exp(-q);
}

// ---- P1: rho per point + partial (sum rho, sum err)
template <typename T, typename TE>
__global__ void __launch_bounds__(kDensThreads) k_dens_rho(const T* __restrict__ tf, int M, int p,
                                                           const T* __restrict__ x, const TE* __restrict__ err,
                                                           int64_t n, double* __restrict__ rho,
                                                           double* __restrict__ part, const TrainCtl* ctl) {
  if (ctl && (ctl->skip || !ctl->density_on)) return;
  extern __shared__ double s_tf[];
  __shared__ double red[32];
  stage_transforms(tf, M, s_tf);
  __syncthreads();
  double srho = 0.0, serr = 0.0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const double x0 = double(x[3 * i]), x1 = double(x[3 * i + 1]), x2 = double(x[3 * i + 2]);
    double r = 0.0;
    for (int m = 0; m < M; ++m) {
      const double* a = s_tf + 13 * m;
      double l0, l1, l2;
      dens_local(a, x0, x1, x2, l0, l1, l2);
      r = add_rn(r, mul_rn(fabs(a[12]), bump_of(l0, l1, l2, p)));
    }
    rho[i] = r;
    srho += r;
    if (err) serr += double(err[i]);
  }
  srho = block_sum(srho, red);
  serr = block_sum(serr, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = srho;
    part[2 * blockIdx.x + 1] = serr;
  }
}

// stats[0] = sum rho, stats[1] = mean err   (single block)
__global__ void k_dens_stats1(const double* __restrict__ part, int nb, int64_t n, double* stats, const TrainCtl* ctl) {
  if (ctl && (ctl->skip || !ctl->density_on)) return;
  __shared__ double red[32];
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) {
    a += part[2 * i];
    b += part[2 * i + 1];
  }
  a = block_sum(a, red);
  b = block_sum(b, red);
  if (threadIdx.x == 0) {
    stats[0] = a;
    stats[1] = b / double(n);
  }
}

// ---- P2: target, loss terms, d_s (density.py:111-148, optim.py:173-177)
template <typename TE>
__global__ void __launch_bounds__(kDensThreads) k_dens_target(const double* __restrict__ rho, const TE* __restrict__ err,
                                                              int64_t n, const double* __restrict__ stats,
                                                              double* __restrict__ d_s, double* __restrict__ part,
                                                              const TrainCtl* ctl) {
  if (ctl && (ctl->skip || !ctl->density_on)) return;
  __shared__ double red[32];
  const double total = stats[0], mean = stats[1];
  const double nn = double(n);
  double sl = 0.0, sd = 0.0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const double rs = div_rn(rho[i], total);
    const double e = double(err[i]);
    const double expo = div_rn(add_rn(mean, kEps), add_rn(e, kEps));
    const double lg = log(add_rn(rs, kEps));
    double star = (expo == 1.0) ? add_rn(rs, kEps) : exp(mul_rn(expo, lg));
    star = fmax(star, kFloor);
    const double ls = log(star);
    sl += mul_rn(rs, sub_rn(lg, ls));
    const double ds = div_rn(add_rn(sub_rn(lg, ls), div_rn(rs, add_rn(rs, kEps))), nn);
    d_s[i] = ds;
    sd += mul_rn(ds, rs);
  }
  sl = block_sum(sl, red);
  sd = block_sum(sd, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = sl;
    part[2 * blockIdx.x + 1] = sd;
  }
}

// stats[2] = loss, stats[3] = sum(d_s * rho_s)
__global__ void k_dens_stats2(const double* __restrict__ part, int nb, int64_t n, double* stats, double* loss,
                              TrainCtl* ctl) {
  if (ctl && (ctl->skip || !ctl->density_on)) return;
  __shared__ double red[32];
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) {
    a += part[2 * i];
    b += part[2 * i + 1];
  }
  a = block_sum(a, red);
  b = block_sum(b, red);
  if (threadIdx.x == 0) {
    stats[2] = a / double(n);
    stats[3] = b;
    if (loss) *loss = a / double(n);
    if (ctl) ctl->l_dens = a / double(n);
  }
}

// ---- P3: per (grid, chunk) gradient accumulators (optim.py:179-195)
// acc[0] = sum w ; acc[1 + 3r + c] = sum s lpow_r x_c ; acc[10 + r] = sum s lpow_r
template <typename T>
__global__ void __launch_bounds__(kDensThreads) k_dens_grad(const T* __restrict__ tf, int M, int p,
                                                            const T* __restrict__ x, int64_t n,
                                                            const double* __restrict__ d_s,
                                                            const double* __restrict__ stats,
                                                            double* __restrict__ part, const TrainCtl* ctl) {
  if (ctl && (ctl->skip || !ctl->density_on)) return;
  __shared__ double red[32];
  __shared__ double a[13];
  const int m = blockIdx.y;
  if (threadIdx.x == 0) {
    double v[12];
    for (int e = 0; e < 12; ++e) v[e] = double(tf[16 * m + e]);
    for (int e = 0; e < 12; ++e) a[e] = v[e];
    const double c0 = sub_rn(mul_rn(v[5], v[10]), mul_rn(v[6], v[9]));
    const double c1 = sub_rn(mul_rn(v[6], v[8]), mul_rn(v[4], v[10]));
    const double c2 = sub_rn(mul_rn(v[4], v[9]), mul_rn(v[5], v[8]));
    a[12] = add_rn(add_rn(mul_rn(v[0], c0), mul_rn(v[2], c2)), mul_rn(v[1], c1));
  }
  __syncthreads();
  const double total = stats[0], S = stats[3], adet = fabs(a[12]);
  double acc[13];
#pragma unroll
  for (int e = 0; e < 13; ++e) acc[e] = 0.0;
  const int64_t chunk = ceil_div(n, int64_t(gridDim.x));
  const int64_t lo = blockIdx.x * chunk, hi = min64(n, lo + chunk);
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const double x0 = double(x[3 * i]), x1 = double(x[3 * i + 1]), x2 = double(x[3 * i + 2]);
    double l0, l1, l2;
    dens_local(a, x0, x1, x2, l0, l1, l2);
    const double s0 = l0 * l0, s1 = l1 * l1, s2 = l2 * l2;
    const double q0 = powi(s0, p - 1), q1 = powi(s1, p - 1), q2 = powi(s2, p - 1);
    const double q = add_rn(add_rn(q0 * s0, q1 * s1), q2 * s2);
    if (!(q <= kClamp)) continue;  // bump == 0 exactly: no contribution (lpow masked, optim.py:189)
    const double bump = exp(-q);
    if (!(bump > 0.0)) continue;
    const double drho = div_rn(sub_rn(d_s[i], S), total);
    const double w = drho * bump;
    const double s = adet * w;
    const double lp0 = l0 * q0, lp1 = l1 * q1, lp2 = l2 * q2;
    acc[0] += w;
    const double sl0 = s * lp0, sl1 = s * lp1, sl2 = s * lp2;
    acc[1] += sl0 * x0;
    acc[2] += sl0 * x1;
    acc[3] += sl0 * x2;
    acc[4] += sl1 * x0;
    acc[5] += sl1 * x1;
    acc[6] += sl1 * x2;
    acc[7] += sl2 * x0;
    acc[8] += sl2 * x1;
    acc[9] += sl2 * x2;
    acc[10] += sl0;
    acc[11] += sl1;
    acc[12] += sl2;
  }
  double* dst = part + (int64_t(blockIdx.x) * M + m) * 13;
#pragma unroll
  for (int e = 0; e < 13; ++e) {
    const double v = block_sum(acc[e], red);
    if (threadIdx.x == 0) dst[e] = v;
  }
}

// ---- P4: per grid: d transforms (optim.py:191-199) [+ masked Adam on the transform group]
template <typename T>
__global__ void k_dens_finalize(T* __restrict__ tf, int M, int p, const double* __restrict__ part, int chunks,
                                T* __restrict__ dtf, T* __restrict__ adam_m, T* __restrict__ adam_v,
                                const TrainCtl* ctl) {
  if (ctl && (ctl->skip || !ctl->density_on)) return;
  __shared__ double red[32];
  const int m = blockIdx.x;  // one block per grid: threads stride over the chunk partials
  double acc[13];
  for (int e = 0; e < 13; ++e) acc[e] = 0.0;
  for (int c = threadIdx.x; c < chunks; c += blockDim.x)
    for (int e = 0; e < 13; ++e) acc[e] += part[(int64_t(c) * M + m) * 13 + e];
  for (int e = 0; e < 13; ++e) acc[e] = block_sum(acc[e], red);
  if (threadIdx.x != 0) return;
  double a[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) a[3 * r + c] = double(tf[16 * m + 4 * r + c]);
  // cofactor rows: a1 x a2, a2 x a0, a0 x a1 (density.py:72-80)
  double cof[9];
  auto cross = [](const double* u, const double* v, double* o) {
    o[0] = sub_rn(mul_rn(u[1], v[2]), mul_rn(u[2], v[1]));
    o[1] = sub_rn(mul_rn(u[2], v[0]), mul_rn(u[0], v[2]));
    o[2] = sub_rn(mul_rn(u[0], v[1]), mul_rn(u[1], v[0]));
  };
  cross(a + 3, a + 6, cof);
  cross(a + 6, a + 0, cof + 3);
  cross(a + 0, a + 3, cof + 6);
  const double det = add_rn(add_rn(mul_rn(a[0], cof[0]), mul_rn(a[2], cof[2])), mul_rn(a[1], cof[1]));
  const double sg = det > 0.0 ? 1.0 : (det < 0.0 ? -1.0 : 0.0);
  const double sw = mul_rn(sg, acc[0]);
  const double twop = 2.0 * double(p);
  T g[16];
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c)
      g[4 * r + c] = T(sub_rn(mul_rn(sw, cof[3 * r + c]), mul_rn(twop, acc[1 + 3 * r + c])));
    g[4 * r + 3] = T(mul_rn(-twop, acc[10 + r]));
  }
  for (int c = 0; c < 4; ++c) g[12 + c] = T(0);
  if (dtf)
    for (int e = 0; e < 16; ++e) dtf[16 * m + e] = g[e];
  if (ctl && adam_m) {  // masked Adam on the transform group (optim.py:47-73, trainer.py:204)
    const T lr = T(ctl->lr_tf_t), c1 = T(ctl->bc1_tf), c2 = T(ctl->bc2_tf);
    for (int e = 0; e < 16; ++e) {
      const T gv = g[e];
      if (gv == T(0)) continue;
      T& mm = adam_m[16 * m + e];
      T& vv = adam_v[16 * m + e];
      mm = add_rn(mul_rn(T(0.9), mm), mul_rn(T(1.0 - 0.9), gv));
      vv = add_rn(mul_rn(T(0.99), vv), mul_rn(T(1.0 - 0.99), mul_rn(gv, gv)));
      const T step = div_rn(mul_rn(lr, div_rn(mm, c1)), add_rn(sqrt_rn(div_rn(vv, c2)), T(1e-8)));
      tf[16 * m + e] = sub_rn(tf[16 * m + e], step);
    }
  }
}

// ---- float-model fast path: the per-(point, grid) bump work in f32 (SFU exp), the
// per-point target/loss pipeline and all reductions in f64.  Bumps below the f32
// range (q > ~87) flush to zero instead of ~1e-38..1e-304; their share of rho and of
// the gradient is below f32 resolution of the sums they enter.
__device__ __forceinline__ void bump32(const float* a, float x0, float x1, float x2, int p, float& bump, float* l,
                                       float* lp) {
  l[0] = fmaf(a[0], x0, fmaf(a[1], x1, fmaf(a[2], x2, a[3])));
  l[1] = fmaf(a[4], x0, fmaf(a[5], x1, fmaf(a[6], x2, a[7])));
  l[2] = fmaf(a[8], x0, fmaf(a[9], x1, fmaf(a[10], x2, a[11])));
  float q = 0.f;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const float s = l[d] * l[d];
    float r;  // s^(p-1)
    if (p == 10) {
      const float s2 = s * s, s4 = s2 * s2, s8 = s4 * s4;
      r = s8 * s;
    } else {
      r = 1.f;
      for (int e = 0; e < p - 1; ++e) r *= s;
    }
    lp[d] = l[d] * r;  // local^(2p-1)
    q = fmaf(r, s, q);
  }
  bump = (q <= 700.f) ? __expf(-q) : 0.f;
}

// bump32 for two points at once in packed fp32x2 (FFMA2 per half = the scalar fmaf), p = 10
// (the flat-top exponent of the APMG models; other p take the scalar kernels).  s = l^2 is
// clamped at 4: a point that far outside has bump exactly 0 either way, and the clamp keeps
// its local^(2p-1) term finite so the packed gradient needs no per-half branch.
__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 f2mul(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 bc2(float v) { return make_float2(v, v); }
__device__ __forceinline__ float ex2_approx(float v) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}
__device__ __forceinline__ void bump32x2(const float* a, float2 x0, float2 x1, float2 x2, float2& bump, float2* l,
                                         float2* lp) {
#pragma unroll
  for (int d = 0; d < 3; ++d)
    l[d] = f2fma(bc2(a[4 * d]), x0, f2fma(bc2(a[4 * d + 1]), x1, f2fma(bc2(a[4 * d + 2]), x2, bc2(a[4 * d + 3]))));
  float2 q = make_float2(0.f, 0.f);
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    float2 s = f2mul(l[d], l[d]);
    s = make_float2(fminf(s.x, 4.f), fminf(s.y, 4.f));
    const float2 s2 = f2mul(s, s), s4 = f2mul(s2, s2), s8 = f2mul(s4, s4);
    const float2 r = f2mul(s8, s);
    lp[d] = f2mul(l[d], r);
    q = f2fma(r, s, q);
  }
  const float2 e = f2mul(q, bc2(-1.4426950408889634f));
  bump = make_float2(ex2_approx(e.x), ex2_approx(e.y));
}

__device__ void stage_transforms32(const float* __restrict__ tf, int M, float* s_tf) {
  for (int m = threadIdx.x; m < M; m += blockDim.x) {
    double a[12];
#pragma unroll
    for (int e = 0; e < 12; ++e) a[e] = double(tf[16 * m + e]);
#pragma unroll
    for (int e = 0; e < 12; ++e) s_tf[13 * m + e] = float(a[e]);
    const double c0 = a[5] * a[10] - a[6] * a[9], c1 = a[6] * a[8] - a[4] * a[10], c2 = a[4] * a[9] - a[5] * a[8];
    s_tf[13 * m + 12] = float(fabs(a[0] * c0 + a[1] * c1 + a[2] * c2));
  }
}

template <typename TE>
__global__ void __launch_bounds__(kDensThreads) k_dens_rho32(const float* __restrict__ tf, int M, int p,
                                                             const float* __restrict__ x, const TE* __restrict__ err,
                                                             int64_t n, double* __restrict__ rho,
                                                             double* __restrict__ part, const TrainCtl* ctl) {
  if (ctl && (ctl->skip || !ctl->density_on)) return;
  extern __shared__ float s_tf32[];
  __shared__ double red[32];
  stage_transforms32(tf, M, s_tf32);
  __syncthreads();
  double srho = 0.0, serr = 0.0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const float x0 = x[3 * i], x1 = x[3 * i + 1], x2 = x[3 * i + 2];
    float r = 0.f;
    for (int m = 0; m < M; ++m) {
      const float* a = s_tf32 + 13 * m;
      float b, l[3], lp[3];
      bump32(a, x0, x1, x2, p, b, l, lp);
      r = fmaf(a[12], b, r);
    }
    rho[i] = double(r);
    srho += double(r);
    if (err) serr += double(err[i]);
  }
  srho = block_sum(srho, red);
  serr = block_sum(serr, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = srho;
    part[2 * blockIdx.x + 1] = serr;
  }
}

// k_dens_rho32 with two consecutive points per thread (p = 10)
// stage_transforms32 with a 16-float stride (16-byte aligned rows)
__device__ void stage_transforms32_16(const float* __restrict__ tf, int M, float* s_tf) {
  for (int m = threadIdx.x; m < M; m += blockDim.x) {
    double a[12];
#pragma unroll
    for (int e = 0; e < 12; ++e) a[e] = double(tf[16 * m + e]);
#pragma unroll
    for (int e = 0; e < 12; ++e) s_tf[16 * m + e] = float(a[e]);
    const double c0 = a[5] * a[10] - a[6] * a[9], c1 = a[6] * a[8] - a[4] * a[10], c2 = a[4] * a[9] - a[5] * a[8];
    s_tf[16 * m + 12] = float(fabs(a[0] * c0 + a[1] * c1 + a[2] * c2));
    s_tf[16 * m + 13] = s_tf[16 * m + 14] = s_tf[16 * m + 15] = 0.f;
  }
}

template <typename TE>
__global__ void __launch_bounds__(kDensThreads) k_dens_rho32x2(const float* __restrict__ tf, int M,
                                                               const float* __restrict__ x,
                                                               const TE* __restrict__ err, int64_t n,
                                                               double* __restrict__ rho, double* __restrict__ part,
                                                               const TrainCtl* ctl) {
  if (ctl && (ctl->skip || !ctl->density_on)) return;
  extern __shared__ float4 s_tf4[];  // [M][4]: rows of A|t, then (det, -, -, -): 4 LDS.128 per grid
  __shared__ double red[32];
  stage_transforms32_16(tf, M, reinterpret_cast<float*>(s_tf4));
  __syncthreads();
  double srho = 0.0, serr = 0.0;
  const int64_t npair = (n + 1) >> 1;
  for (int64_t ip = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; ip < npair;
       ip += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = 2 * ip;
    const bool two = i + 1 < n;
    float2 X0, X1, X2;
    if (two) {
      const float2* xp = reinterpret_cast<const float2*>(x + 3 * i);
      const float2 f0 = xp[0], f1 = xp[1], f2 = xp[2];
      X0 = make_float2(f0.x, f1.y);
      X1 = make_float2(f0.y, f2.x);
      X2 = make_float2(f1.x, f2.y);
    } else {
      X0 = bc2(x[3 * i]);
      X1 = bc2(x[3 * i + 1]);
      X2 = bc2(x[3 * i + 2]);
    }
    float2 r = make_float2(0.f, 0.f);
#pragma unroll 2
    for (int m = 0; m < M; ++m) {
      const float4 t0 = s_tf4[4 * m], t1 = s_tf4[4 * m + 1], t2 = s_tf4[4 * m + 2], t3 = s_tf4[4 * m + 3];
      const float a[13] = {t0.x, t0.y, t0.z, t0.w, t1.x, t1.y, t1.z, t1.w, t2.x, t2.y, t2.z, t2.w, t3.x};
      float2 b, l[3], lp[3];
      bump32x2(a, X0, X1, X2, b, l, lp);
      r = f2fma(bc2(a[12]), b, r);
    }
    rho[i] = double(r.x);
    srho += double(r.x);
    if (err) serr += double(err[i]);
    if (two) {
      rho[i + 1] = double(r.y);
      srho += double(r.y);
      if (err) serr += double(err[i + 1]);
    }
  }
  srho = block_sum(srho, red);
  serr = block_sum(serr, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = srho;
    part[2 * blockIdx.x + 1] = serr;
  }
}

// d_rho = (d_s - sum(d_s rho_s)) / sum(rho) per point, once (optim.py:182-183), as f32
__global__ void k_dens_drho32(const double* __restrict__ d_s, int64_t n, const double* __restrict__ stats,
                              float* __restrict__ drho, const TrainCtl* ctl) {
  if (ctl && (ctl->skip || !ctl->density_on)) return;
  const double total = stats[0], S = stats[3];
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    drho[i] = float((d_s[i] - S) / total);
}

__global__ void __launch_bounds__(kDensThreads) k_dens_grad32(const float* __restrict__ tf, int M, int p,
                                                              const float* __restrict__ x, int64_t n,
                                                              const float* __restrict__ drho,
                                                              double* __restrict__ part, const TrainCtl* ctl) {
  if (ctl && (ctl->skip || !ctl->density_on)) return;
  __shared__ double red[32];
  __shared__ float a[13];
  const int m = blockIdx.y;
  if (threadIdx.x == 0) stage_transforms32(tf + 16 * m, 1, a);
  __syncthreads();
  const float adet = a[12];
  float acc[13];
#pragma unroll
  for (int e = 0; e < 13; ++e) acc[e] = 0.f;
  const int64_t chunk = ceil_div(n, int64_t(gridDim.x));
  const int64_t lo = blockIdx.x * chunk, hi = min64(n, lo + chunk);
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const float x0 = x[3 * i], x1 = x[3 * i + 1], x2 = x[3 * i + 2];
    float b, l[3], lp[3];
    bump32(a, x0, x1, x2, p, b, l, lp);
    if (!(b > 0.f)) continue;
    const float w = drho[i] * b;
    const float s = adet * w;
    acc[0] += w;
    const float sl0 = s * lp[0], sl1 = s * lp[1], sl2 = s * lp[2];
    acc[1] = fmaf(sl0, x0, acc[1]);
    acc[2] = fmaf(sl0, x1, acc[2]);
    acc[3] = fmaf(sl0, x2, acc[3]);
    acc[4] = fmaf(sl1, x0, acc[4]);
    acc[5] = fmaf(sl1, x1, acc[5]);
    acc[6] = fmaf(sl1, x2, acc[6]);
    acc[7] = fmaf(sl2, x0, acc[7]);
    acc[8] = fmaf(sl2, x1, acc[8]);
    acc[9] = fmaf(sl2, x2, acc[9]);
    acc[10] += sl0;
    acc[11] += sl1;
    acc[12] += sl2;
  }
  double* dst = part + (int64_t(blockIdx.x) * M + m) * 13;
#pragma unroll
  for (int e = 0; e < 13; ++e) {
    const double v = block_sum(double(acc[e]), red);
    if (threadIdx.x == 0) dst[e] = v;
  }
}

// Chunked variant: a block stages kGradCH points (x, d_rho) in shared memory once and its
// warps sweep them for every grid (the per-grid launch above re-reads x and d_rho M times);
// per-(chunk, grid) lane sums are combined in f64 per block.
constexpr int kGradCH = 4096;
constexpr int kGradMaxM = 128;
__global__ void __launch_bounds__(kDensThreads) k_dens_grad32c(const float* __restrict__ tf, int M, int p,
                                                               const float* __restrict__ x, int64_t n,
                                                               const float* __restrict__ drho, int ch,
                                                               double* __restrict__ part, const TrainCtl* ctl) {
  if (ctl && (ctl->skip || !ctl->density_on)) return;
  extern __shared__ float4 sP[];                                   // [ch <= kGradCH] (x0, x1, x2, d_rho)
  double* s_acc = reinterpret_cast<double*>(sP + kGradCH);         // [M][13]
  float* s_tf = reinterpret_cast<float*>(s_acc + 13 * M);          // [M][13]
  stage_transforms32(tf, M, s_tf);
  for (int e = threadIdx.x; e < 13 * M; e += blockDim.x) s_acc[e] = 0.0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int64_t c0 = int64_t(blockIdx.x) * ch; c0 < n; c0 += int64_t(gridDim.x) * ch) {
    const int cnt = int(min64(ch, n - c0));
    __syncthreads();  // previous chunk consumed, transforms / accumulators staged
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
      const int64_t g = c0 + i;
      sP[i] = make_float4(x[3 * g], x[3 * g + 1], x[3 * g + 2], drho[g]);
    }
    __syncthreads();
    for (int m = warp; m < M; m += nw) {
      float a[13];
#pragma unroll
      for (int e = 0; e < 13; ++e) a[e] = s_tf[13 * m + e];
      float acc[13];
#pragma unroll
      for (int e = 0; e < 13; ++e) acc[e] = 0.f;
      for (int i = lane; i < cnt; i += 32) {
        const float4 q = sP[i];
        float b, l[3], lp[3];
        bump32(a, q.x, q.y, q.z, p, b, l, lp);
        if (!(b > 0.f)) continue;
        const float w = q.w * b;
        const float sc = a[12] * w;
        acc[0] += w;
        const float sl0 = sc * lp[0], sl1 = sc * lp[1], sl2 = sc * lp[2];
        acc[1] = fmaf(sl0, q.x, acc[1]);
        acc[2] = fmaf(sl0, q.y, acc[2]);
        acc[3] = fmaf(sl0, q.z, acc[3]);
        acc[4] = fmaf(sl1, q.x, acc[4]);
        acc[5] = fmaf(sl1, q.y, acc[5]);
        acc[6] = fmaf(sl1, q.z, acc[6]);
        acc[7] = fmaf(sl2, q.x, acc[7]);
        acc[8] = fmaf(sl2, q.y, acc[8]);
        acc[9] = fmaf(sl2, q.z, acc[9]);
        acc[10] += sl0;
        acc[11] += sl1;
        acc[12] += sl2;
      }
#pragma unroll
      for (int e = 0; e < 13; ++e) {
        const double v = warp_sum(double(acc[e]));
        if (lane == 0) s_acc[13 * m + e] += v;
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 13 * M; e += blockDim.x) part[int64_t(blockIdx.x) * 13 * M + e] = s_acc[e];
}

// k_dens_grad32c with two staged points per lane and step (p = 10): float2 accumulators
__global__ void __launch_bounds__(kDensThreads, 2) k_dens_grad32cx2(const float* __restrict__ tf, int M,
                                                                 const float* __restrict__ x, int64_t n,
                                                                 const double* __restrict__ d_s,
                                                                 const double* __restrict__ stats, int ch,
                                                                 double* __restrict__ part, const TrainCtl* ctl) {
  if (ctl && (ctl->skip || !ctl->density_on)) return;
  // the chunk's points as lane pairs (i, i + 32) of each 64-point run, pre-paired so that the packed
  // fp32x2 arithmetic reads its operand pairs straight from two 16-byte loads:
  // sP[2 j] = (x0_a, x0_b, x1_a, x1_b), sP[2 j + 1] = (x2_a, x2_b, d_rho_a, d_rho_b)
  extern __shared__ float4 sP[];                                   // [ch <= kGradCH] (2 float4 per pair)
  const double total = stats[0], S = stats[3];  // d_rho formed while staging (k_dens_drho32's value)
  double* s_acc = reinterpret_cast<double*>(sP + kGradCH);         // [M][13]
  float* s_tf = reinterpret_cast<float*>(s_acc + 13 * M);          // [M][13]
  stage_transforms32(tf, M, s_tf);
  for (int e = threadIdx.x; e < 13 * M; e += blockDim.x) s_acc[e] = 0.0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int64_t c0 = int64_t(blockIdx.x) * ch; c0 < n; c0 += int64_t(gridDim.x) * ch) {
    const int cnt = int(min64(ch, n - c0));
    __syncthreads();  // previous chunk consumed, transforms / accumulators staged
    float* sF = reinterpret_cast<float*>(sP);
    for (int i = threadIdx.x; i < ((cnt + 63) & ~63); i += blockDim.x) {
      const int64_t g = c0 + i;
      const bool ok = i < cnt;  // d_rho 0 past the end: no share
      const int j = (i >> 6) * 32 + (i & 31), h = (i >> 5) & 1;
      sF[8 * j + h] = ok ? x[3 * g] : 0.f;
      sF[8 * j + 2 + h] = ok ? x[3 * g + 1] : 0.f;
      sF[8 * j + 4 + h] = ok ? x[3 * g + 2] : 0.f;
      sF[8 * j + 6 + h] = ok ? float((d_s[g] - S) / total) : 0.f;
    }
    __syncthreads();
    // two grids per pass (m, m + nw): independent chains for the scheduler, one read of the points
    for (int m = warp; m < M; m += 2 * nw) {
      const int m2 = m + nw;
      const bool two = m2 < M;
      float a[2][13];
#pragma unroll
      for (int e = 0; e < 13; ++e) {
        a[0][e] = s_tf[13 * m + e];
        a[1][e] = two ? s_tf[13 * m2 + e] : 0.f;
      }
      float2 acc[2][13];
#pragma unroll
      for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int e = 0; e < 13; ++e) acc[k][e] = make_float2(0.f, 0.f);
      for (int i = lane; i < cnt; i += 64) {
        const int j = (i >> 6) * 32 + lane;
        const float4 q0 = sP[2 * j], q1 = sP[2 * j + 1];
        const float2 X0 = make_float2(q0.x, q0.y), X1 = make_float2(q0.z, q0.w), X2 = make_float2(q1.x, q1.y);
        const float2 W = make_float2(q1.z, q1.w);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          float2 b, l[3], lp[3];
          bump32x2(a[k], X0, X1, X2, b, l, lp);
          const float2 w = f2mul(W, b);
          const float2 sc = f2mul(bc2(a[k][12]), w);
          acc[k][0] = __fadd2_rn(acc[k][0], w);
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            const float2 sl = f2mul(sc, lp[d]);
            acc[k][1 + 3 * d] = f2fma(sl, X0, acc[k][1 + 3 * d]);
            acc[k][2 + 3 * d] = f2fma(sl, X1, acc[k][2 + 3 * d]);
            acc[k][3 + 3 * d] = f2fma(sl, X2, acc[k][3 + 3 * d]);
            acc[k][10 + d] = __fadd2_rn(acc[k][10 + d], sl);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        if (k == 1 && !two) break;
        const int mk = k ? m2 : m;
#pragma unroll
        for (int e = 0; e < 13; ++e) {
          const double v = warp_sum(double(acc[k][e].x) + double(acc[k][e].y));
          if (lane == 0) s_acc[13 * mk + e] += v;
        }
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 13 * M; e += blockDim.x) part[int64_t(blockIdx.x) * 13 * M + e] = s_acc[e];
}

static size_t grad32c_smem(int M) { return sizeof(float4) * kGradCH + size_t(13) * M * (sizeof(double) + sizeof(float)); }

struct DensPlan {
  int nb1, chunks, nbg;  // nbg: blocks of the chunked f32 gradient kernel
};

static DensPlan dens_plan(int M, int64_t n) {
  DensPlan d;
  d.nb1 = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, kDensThreads), int64_t(num_sms()) * 8)));
  const int64_t want = std::max<int64_t>(1, (int64_t(num_sms()) * 8 + M - 1) / M);
  d.chunks = int(std::max<int64_t>(1, std::min<int64_t>(want, ceil_div(n, kDensThreads))));
  d.nbg = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 512), int64_t(num_sms()) * 2)));
  return d;
}

size_t density_ws_bytes(int M, int64_t n) {
  DensPlan d = dens_plan(M, n);
  Carver c(nullptr, 0);
  c.take<double>(n);                          // rho
  c.take<double>(n);                          // d_s
  c.take<double>(2 * size_t(std::max(d.nb1, num_sms())));  // part1 (or the fused recon's per-CTA sums)
  c.take<double>(2 * size_t(d.nb1));          // part2
  c.take<double>(size_t(std::max(d.chunks, d.nbg)) * M * 13);  // part3
  c.take<double>(8);                                             // stats
  return c.used + 256;
}

static bool packed_density() {  // APMG_DENSITY_X2=0: the one-point-per-lane kernels (A/B)
  const char* e = getenv("APMG_DENSITY_X2");
  return !(e && e[0] == '0');
}

int density_rho_slots(int M, int64_t n, void* ws, size_t wsb, double** rho, double** part1) {
  DensPlan d = dens_plan(M, n);
  Carver c(ws, wsb);
  *rho = c.take<double>(n);
  c.take<double>(n);
  *part1 = c.take<double>(2 * size_t(std::max(d.nb1, num_sms())));
  if (!c.ok()) {
    set_error("density workspace too small: need %zu, have %zu", c.used, wsb);
    return APMG_E_WORKSPACE;
  }
  return APMG_OK;
}

template <typename T, typename TE>
int launch_density(T* tf, int M, int p, const T* x, const TE* err, int64_t n, double* loss, T* dtf,
                   double* rho_total, T* adam_m, T* adam_v, void* ws, size_t wsb, const TrainCtl* ctl,
                   cudaStream_t st, int pre_nb) {
  APMG_ARG_CHECK(M <= kMaxGridsSmem, "density supports up to %d grids", kMaxGridsSmem);
  DensPlan d = dens_plan(M, n);
  Carver c(ws, wsb);
  double* rho = c.take<double>(n);
  double* d_s = c.take<double>(n);
  double* part1 = c.take<double>(2 * size_t(std::max(d.nb1, num_sms())));
  double* part2 = c.take<double>(2 * size_t(d.nb1));
  double* part3 = c.take<double>(size_t(std::max(d.chunks, d.nbg)) * M * 13);
  double* stats = c.take<double>(8);
  if (!c.ok()) {
    set_error("density workspace too small: need %zu, have %zu", c.used, wsb);
    return APMG_E_WORKSPACE;
  }
  int parts = d.chunks;  // gradient partials per grid handed to the finalize kernel
  const char* e64 = getenv("APMG_DENSITY64");  // force the all-fp64 per-pair path (A/B tests)
  const bool fast32 = (sizeof(T) == 4) && !(e64 && e64[0] == '1');
  APMG_ARG_CHECK(!pre_nb || (fast32 && p == 10), "a precomputed rho needs the f32 p = 10 density path");
  if constexpr (sizeof(T) == 4) {
    if (fast32 && !pre_nb) {
      const size_t smem32 = size_t(13) * M * sizeof(float);
      APMG_CUDA_TRY(
          cudaFuncSetAttribute(k_dens_rho32<TE>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem32)));
      if (p == 10 && packed_density()) {
        const size_t smem16 = size_t(16) * M * sizeof(float);
        APMG_CUDA_TRY(
            cudaFuncSetAttribute(k_dens_rho32x2<TE>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem16)));
        APMG_LAUNCH("density_rho", k_dens_rho32x2<TE>, d.nb1, kDensThreads, smem16, st, tf, M, x, err, n, rho, part1,
                    ctl);
      } else {
        APMG_LAUNCH("density_rho", k_dens_rho32<TE>, d.nb1, kDensThreads, smem32, st, tf, M, p, x, err, n, rho,
                    part1, ctl);
      }
    }
  }
  if (!fast32) {
    const size_t smem1 = size_t(13) * M * sizeof(double);
    APMG_CUDA_TRY(cudaFuncSetAttribute(k_dens_rho<T, TE>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem1)));
    APMG_LAUNCH("density_rho", (k_dens_rho<T, TE>), d.nb1, kDensThreads, smem1, st, tf, M, p, x, err, n, rho, part1,
                ctl);
  }
  APMG_LAUNCH("density_stats", k_dens_stats1, 1, 1024, 0, st, part1, pre_nb ? pre_nb : d.nb1, n, stats, ctl);
  APMG_LAUNCH("density_target", k_dens_target<TE>, d.nb1, kDensThreads, 0, st, rho, err, n, stats, d_s, part2, ctl);
  APMG_LAUNCH("density_stats", k_dens_stats2, 1, 1024, 0, st, part2, d.nb1, n, stats, loss,
              const_cast<TrainCtl*>(ctl));
  if constexpr (sizeof(T) == 4) {
    if (fast32) {
      float* drho = reinterpret_cast<float*>(rho);  // rho is dead once the target pass has run
      const bool x2 = M <= kGradMaxM && p == 10 && packed_density();  // forms d_rho itself
      if (!x2) APMG_LAUNCH("density_drho", k_dens_drho32, d.nb1, kDensThreads, 0, st, d_s, n, stats, drho, ctl);
      if (M <= kGradMaxM) {
        const size_t sm = grad32c_smem(M);
        const int ch = int(std::min<int64_t>(kGradCH, ceil_div(n, d.nbg)));  // one balanced chunk per block
        if (p == 10 && packed_density()) {
          APMG_CUDA_TRY(
              cudaFuncSetAttribute(k_dens_grad32cx2, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
          APMG_LAUNCH("density_grad", k_dens_grad32cx2, d.nbg, kDensThreads, sm, st, tf, M, x, n, d_s, stats, ch,
                      part3, ctl);
        } else {
          APMG_CUDA_TRY(cudaFuncSetAttribute(k_dens_grad32c, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
          APMG_LAUNCH("density_grad", k_dens_grad32c, d.nbg, kDensThreads, sm, st, tf, M, p, x, n, drho, ch, part3,
                      ctl);
        }
        parts = d.nbg;
      } else {
        APMG_LAUNCH("density_grad", k_dens_grad32, dim3(d.chunks, M), kDensThreads, 0, st, tf, M, p, x, n, drho,
                    part3, ctl);
      }
    }
  }
  if (!fast32)
    APMG_LAUNCH("density_grad", k_dens_grad<T>, dim3(d.chunks, M), kDensThreads, 0, st, tf, M, p, x, n, d_s, stats,
                part3, ctl);
  APMG_LAUNCH("density_finalize", k_dens_finalize<T>, M, 128, 0, st, tf, M, p, part3, parts, dtf, adam_m, adam_v,
              ctl);
  if (rho_total) APMG_CUDA_TRY(cudaMemcpyAsync(rho_total, stats, sizeof(double), cudaMemcpyDeviceToDevice, st));
  return APMG_OK;
}

template int launch_density<float, float>(float*, int, int, const float*, const float*, int64_t, double*, float*,
                                          double*, float*, float*, void*, size_t, const TrainCtl*, cudaStream_t, int);
template int launch_density<double, double>(double*, int, int, const double*, const double*, int64_t, double*,
                                            double*, double*, double*, double*, void*, size_t, const TrainCtl*,
                                            cudaStream_t, int);

// ---- standalone elementwise helpers
__global__ void k_feature_density_f64pts(const double* __restrict__ s_tf_g, int M, int p, const double* __restrict__ x,
                                         int64_t n, double* __restrict__ rho) {
  extern __shared__ double s_tf[];
  for (int e = threadIdx.x; e < 13 * M; e += blockDim.x) s_tf[e] = s_tf_g[e];
  __syncthreads();
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    double r = 0.0;
    for (int m = 0; m < M; ++m) {
      const double* a = s_tf + 13 * m;
      double l0, l1, l2;
      dens_local(a, x[3 * i], x[3 * i + 1], x[3 * i + 2], l0, l1, l2);
      r = add_rn(r, mul_rn(fabs(a[12]), bump_of(l0, l1, l2, p)));
    }
    rho[i] = r;
  }
}

template <typename T>
__global__ void k_stage_tf(const T* __restrict__ tf, int M, double* out) {
  extern __shared__ double s[];
  stage_transforms(tf, M, s);
  __syncthreads();
  for (int e = threadIdx.x; e < 13 * M; e += blockDim.x) out[e] = s[e];
}

__global__ void k_target(const double* __restrict__ rs, const double* __restrict__ err, int64_t n, double mean,
                         double eps, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const double expo = div_rn(add_rn(mean, eps), add_rn(err[i], eps));
    const double v = (expo == 1.0) ? add_rn(rs[i], eps) : exp(mul_rn(expo, log(add_rn(rs[i], eps))));
    out[i] = fmax(v, kFloor);
  }
}

__global__ void k_loss_terms(const double* __restrict__ rs, const double* __restrict__ star, int64_t n, double eps,
                             double* __restrict__ out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = mul_rn(rs[i], sub_rn(log(add_rn(rs[i], eps)), log(star[i])));
}

__global__ void k_scale(const double* __restrict__ x, int64_t n, const double* __restrict__ div,
                        double* __restrict__ out) {
  const double d = *div;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = div_rn(x[i], d);
}

__global__ void k_sum_partial(const double* __restrict__ x, int64_t n, double* __restrict__ part) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    s += x[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void k_sum_final(const double* __restrict__ part, int nb, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) s += part[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s;
}

static int elt_grid(int64_t n) {
  return int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), int64_t(num_sms()) * 8)));
}

}  // namespace apmg

using namespace apmg;

extern "C" size_t apmg_density_workspace_bytes(int32_t grids, int64_t n) { return density_ws_bytes(grids, n); }

extern "C" int apmg_density_loss_grads(const apmg_model* m, const void* coords, const double* errors, int64_t n,
                                       double* loss, void* d_transforms, double* rho_total, void* workspace,
                                       size_t workspace_bytes, void* stream) {
  APMG_ARG_CHECK(m && (m->dtype == APMG_F32 || m->dtype == APMG_F64), "bad model");
  APMG_ARG_CHECK(n >= 2, "density batch needs >= 2 coordinates with matching errors");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // the host wrapper passes errors as f64 (optim.py:167); the transforms are only read here
  if (m->dtype == APMG_F32) {
    return launch_density<float, double>(const_cast<float*>(static_cast<const float*>(m->transforms)), m->grids,
                                         m->flat_top_p, static_cast<const float*>(coords), errors, n, loss,
                                         static_cast<float*>(d_transforms), rho_total, nullptr, nullptr, workspace,
                                         workspace_bytes, nullptr, st);
  }
  return launch_density<double, double>(const_cast<double*>(static_cast<const double*>(m->transforms)), m->grids,
                                        m->flat_top_p, static_cast<const double*>(coords), errors, n, loss,
                                        static_cast<double*>(d_transforms), rho_total, nullptr, nullptr, workspace,
                                        workspace_bytes, nullptr, st);
}

extern "C" int apmg_feature_density(int32_t dtype, const void* transforms, int32_t grids, int32_t p,
                                    const double* pts, int64_t n, double* rho, void* stream) {
  APMG_ARG_CHECK(grids >= 1 && grids <= kMaxGridsSmem, "bad grid count");
  APMG_ARG_CHECK(p >= 1, "flat-top strength p must be >= 1");
  if (n <= 0) return APMG_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* staged = nullptr;
  APMG_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&staged), sizeof(double) * 13 * grids, st));
  const size_t smem = sizeof(double) * 13 * grids;
  if (dtype == APMG_F32)
    APMG_LAUNCH("stage_tf", k_stage_tf<float>, 1, 128, smem, st, static_cast<const float*>(transforms), grids, staged);
  else
    APMG_LAUNCH("stage_tf", k_stage_tf<double>, 1, 128, smem, st, static_cast<const double*>(transforms), grids,
                staged);
  APMG_CUDA_TRY(cudaFuncSetAttribute(k_feature_density_f64pts, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  APMG_LAUNCH("feature_density", k_feature_density_f64pts, elt_grid(n), 256, smem, st, staged, grids, p, pts, n, rho);
  APMG_CUDA_TRY(cudaFreeAsync(staged, st));
  return APMG_OK;
}

extern "C" int apmg_target_density(const double* rho_scaled, const double* errors, int64_t n, double mean_error,
                                   double eps, double* rho_star, void* stream) {
  if (n <= 0) return APMG_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  APMG_LAUNCH("target_density", k_target, elt_grid(n), 256, 0, st, rho_scaled, errors, n, mean_error, eps, rho_star);
  return APMG_OK;
}

extern "C" int apmg_density_loss_terms(const double* rho_scaled, const double* rho_star, int64_t n, double eps,
                                       double* terms, void* stream) {
  if (n <= 0) return APMG_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  APMG_LAUNCH("density_loss_terms", k_loss_terms, elt_grid(n), 256, 0, st, rho_scaled, rho_star, n, eps, terms);
  return APMG_OK;
}

extern "C" int apmg_scale_f64(const double* x, int64_t n, const double* divisor, double* out, void* stream) {
  if (n <= 0) return APMG_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  APMG_LAUNCH("scale", k_scale, elt_grid(n), 256, 0, st, x, n, divisor, out);
  return APMG_OK;
}

extern "C" size_t apmg_sum_workspace_bytes(int64_t n) { return sizeof(double) * (elt_grid(n) + 1) + 256; }

extern "C" int apmg_sum_f64(const double* x, int64_t n, double* out, void* workspace, size_t workspace_bytes,
                            void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int nb = elt_grid(std::max<int64_t>(n, 1));
  if (workspace_bytes < sizeof(double) * nb) {
    set_error("sum workspace too small");
    return APMG_E_WORKSPACE;
  }
  double* part = static_cast<double*>(workspace);
  APMG_LAUNCH("sum_partial", k_sum_partial, nb, 256, 0, st, x, n, part);
  APMG_LAUNCH("sum_final", k_sum_final, 1, 1024, 0, st, part, nb, out);
  return APMG_OK;
}

// feature_density_terms (density.py:83-103): local (M,N,3), dets (M), bumps (M,N), rho (N), all f64.
namespace apmg {
__global__ void k_density_terms(const double* __restrict__ staged, int M, int p, const double* __restrict__ x,
                                int64_t n, double* __restrict__ local, double* __restrict__ bumps) {
  const int64_t total = int64_t(M) * n;
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < total; q += int64_t(gridDim.x) * blockDim.x) {
    const int m = int(q / n);
    const int64_t i = q - int64_t(m) * n;
    const double* a = staged + 13 * m;
    double l0, l1, l2;
    dens_local(a, x[3 * i], x[3 * i + 1], x[3 * i + 2], l0, l1, l2);
    local[3 * q] = l0;
    local[3 * q + 1] = l1;
    local[3 * q + 2] = l2;
    bumps[q] = bump_of(l0, l1, l2, p);
  }
}
__global__ void k_dets(const double* __restrict__ staged, int M, double* dets) {
  for (int m = threadIdx.x; m < M; m += blockDim.x) dets[m] = staged[13 * m + 12];
}
}  // namespace apmg

extern "C" int apmg_density_terms(int32_t dtype, const void* transforms, int32_t grids, int32_t p, const double* pts,
                                  int64_t n, double* local, double* dets, double* bumps, double* rho, void* stream) {
  APMG_ARG_CHECK(grids >= 1 && grids <= kMaxGridsSmem, "bad grid count");
  APMG_ARG_CHECK(p >= 1, "flat-top strength p must be >= 1");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* staged = nullptr;
  APMG_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&staged), sizeof(double) * 13 * grids, st));
  const size_t smem = sizeof(double) * 13 * grids;
  if (dtype == APMG_F32)
    APMG_LAUNCH("stage_tf", k_stage_tf<float>, 1, 128, smem, st, static_cast<const float*>(transforms), grids, staged);
  else
    APMG_LAUNCH("stage_tf", k_stage_tf<double>, 1, 128, smem, st, static_cast<const double*>(transforms), grids,
                staged);
  APMG_LAUNCH("dets", k_dets, 1, 128, 0, st, staged, grids, dets);
  if (n > 0) {
    APMG_LAUNCH("density_terms", k_density_terms, elt_grid(int64_t(grids) * n), 256, 0, st, staged, grids, p, pts, n,
                local, bumps);
    APMG_CUDA_TRY(
        cudaFuncSetAttribute(k_feature_density_f64pts, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    APMG_LAUNCH("feature_density", k_feature_density_f64pts, elt_grid(n), 256, smem, st, staged, grids, p, pts, n,
                rho);
  }
  APMG_CUDA_TRY(cudaFreeAsync(staged, st));
  return APMG_OK;
}
