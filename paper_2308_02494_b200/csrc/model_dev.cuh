// Device view of an APMGSRN model and the per-(point, grid) encoder primitives.
//
// Numerics follow the reference exactly where it is elementwise numpy:
//  * to_local (model.py:179-182): numpy einsum("nk,ok->no") sums the 3 products
//    as (p0a0 + p1a1) + p2a2 for float32 and (p0a0 + p2a2) + p1a1 for float64,
//    each product/sum rounded separately (pinned in tests/test_oracle.py).
//  * grid_interp_terms (model.py:198-213): u = ((l + 1) * 0.5) * (n - 1) in the
//    model dtype, i0 = clip(floor(u), 0, n-2), frac = clip(f64(u) - i0, 0, 1).
//  * _interp_channels (model.py:216-226): lerp a + f*(b - a) where (b - a) is
//    rounded in the model dtype and everything after it is float64; the
//    result is rounded to the model dtype.
//  * backward weights (optim.py:129-152): w = (wx * wy) * wz in f64.
#pragma once
#ifndef APMG_AGG_ROUNDS
#define APMG_AGG_ROUNDS 2  // tree rounds cap: groups above 4 lanes issue one RED set per 4-lane block
                          // (3 rounds measured 3% faster than the full 5: shuffles are the bound)
#endif

#include "common.cuh"

namespace apmg {

// fixed-point scale of the deterministic grid gradient: 2^44 (resolution 5.7e-14, range +-5.2e5)
constexpr double kFxScale = 17592186044416.0, kFxInv = 1.0 / 17592186044416.0;
__device__ __forceinline__ void red_fx(unsigned long long* addr, double v) {
  atomicAdd(addr, static_cast<unsigned long long>(__double2ll_rn(v * kFxScale)));
}
// the same for a float: v * 2^44 is exact in float, so rounding it to int64 there gives the double
// path's integer without the f64 conversions
__device__ __forceinline__ void red_fx(unsigned long long* addr, float v) {
  atomicAdd(addr, static_cast<unsigned long long>(__float2ll_rn(v * 17592186044416.0f)));
}

template <typename T>
struct ModelDev {
  int M, C, D, H, W, F, p;
  const T* __restrict__ tf;    // [M][4][4]
  const T* __restrict__ grid;  // [M][D][H][W][C]
  const T* __restrict__ w1;    // [64][F]
  const T* __restrict__ w2;    // [64][64]
  const T* __restrict__ w3;    // [64]
  T span, vmin;                // np.asarray(vmax - vmin, dtype), np.asarray(vmin, dtype)
  // optional x-pair copy of a two-channel f32 grid (training sessions): gridx[c] =
  // (grid[c], grid[c + 1]) over the flat cell index c, so the two x-corners of a cell edge
  // are one 16-byte load -- the encoder's gathers are L2-request-bound, not byte-bound
  const float4* __restrict__ gridx = nullptr;
  // or the xy-quad copy (32 bytes per cell c: grid[c], grid[c + 1], grid[c + W], grid[c + W + 1]),
  // so a cell's four corners of one z plane are one 256-bit load (2 gathers per (point, grid))
  const float* __restrict__ gridq = nullptr;
  // the grid gradient the recon kernel scatters into is in the same x-pair layout
  // (dgridx[c] = d/d(grid[c]), d/d(grid[c + 1]) partial sums; float4 REDs, half the RED
  // operations): grad(grid[v]) = dgridx[v].lo + dgridx[v - 1].hi.  tc16 kernel only.
  bool grad_pairs = false;
  // deterministic training: the grid gradient is accumulated as 64-bit fixed point (kFxScale)
  // with integer REDs -- associative, so the sum is independent of arrival order
  unsigned long long* dgrid_fx = nullptr;
  // fused density pass (training, f32, p = 10; tc16 kernel only): the encoder's local
  // coordinates also give the flat-top bumps, so the kernel writes rho per point
  // (density.py:83-103) and per-CTA (sum rho, sum sq_err) partials -- the density step then
  // starts at its statistics (optim.py:158-200)
  double* rho_out = nullptr;
  double* rho_part = nullptr;
};

template <typename T>
inline ModelDev<T> make_model_dev(const apmg_model& m) {
  ModelDev<T> d;
  d.M = m.grids;
  d.C = m.channels;
  d.D = m.depth;
  d.H = m.height;
  d.W = m.width;
  d.F = m.grids * m.channels;
  d.p = m.flat_top_p;
  d.tf = static_cast<const T*>(m.transforms);
  d.grid = static_cast<const T*>(m.grids_cl);
  d.w1 = static_cast<const T*>(m.w1);
  d.w2 = static_cast<const T*>(m.w2);
  d.w3 = static_cast<const T*>(m.w3);
  d.span = static_cast<T>(m.vmax - m.vmin);
  d.vmin = static_cast<T>(m.vmin);
  return d;
}

__device__ __forceinline__ float local_coord(float x0, float x1, float x2, float a0, float a1, float a2,
                                             float t) {
  return add_rn(add_rn(add_rn(mul_rn(x0, a0), mul_rn(x1, a1)), mul_rn(x2, a2)), t);
}
__device__ __forceinline__ double local_coord(double x0, double x1, double x2, double a0, double a1,
                                              double a2, double t) {
  return add_rn(add_rn(add_rn(mul_rn(x0, a0), mul_rn(x2, a2)), mul_rn(x1, a1)), t);
}

// local_coord<float> for two points at once: scalar products, packed sums (FADD2, each half
// rounded as the scalar add).  The products stay scalar on purpose: ptxas (CUDA 12.9)
// contracts mul.rn.f32x2 + add.rn.f32x2 into FFMA2 despite the explicit rounding modifiers,
// which would change the rounding of the local coordinates (and flip inside/outside tests).
__device__ __forceinline__ float2 mul_s2(float2 x, float a) { return make_float2(__fmul_rn(x.x, a), __fmul_rn(x.y, a)); }
__device__ __forceinline__ float2 local_coord2(float2 x0, float2 x1, float2 x2, float a0, float a1, float a2,
                                               float t) {
  const float2 p = __fadd2_rn(__fadd2_rn(mul_s2(x0, a0), mul_s2(x1, a1)), mul_s2(x2, a2));
  return __fadd2_rn(p, make_float2(t, t));
}

// Interpolation terms of one point in one grid.
struct Cell {
  int ix, iy, iz;
  double fx, fy, fz;
  bool inside;
};

// numpy: i0 = clip(floor(u), 0, n-2), frac = clip(f64(u) - i0, 0, 1).  For points inside
// the grid u lies in [0, n-1], so both clips are no-ops except i0 at the top vertex, and
// u - i0 is exact in the model dtype (Sterbenz), hence computed there.  Outside points
// only need an in-range index (their features are zeroed / their scatter is skipped).
__device__ __forceinline__ void axis_term(float l, int n, int& i0, double& f) {
  const float u = mul_rn(mul_rn(add_rn(l, 1.0f), 0.5f), float(n - 1));
  const int i = min(max(int(floorf(u)), 0), n - 2);
  i0 = i;
  f = static_cast<double>(__fsub_rn(u, float(i)));
}
// axis_term<float> for two points: (l + 1) * 0.5 packed, the rest scalar (see local_coord2:
// a packed multiply feeding the fraction's subtraction would be contracted)
__device__ __forceinline__ void axis_term2(float2 l, int n, int& i0, int& i1, float& f0, float& f1) {
  const float2 h = __fmul2_rn(__fadd2_rn(l, make_float2(1.0f, 1.0f)), make_float2(0.5f, 0.5f));
  const float u0 = __fmul_rn(h.x, float(n - 1)), u1 = __fmul_rn(h.y, float(n - 1));
  i0 = min(max(int(floorf(u0)), 0), n - 2);
  i1 = min(max(int(floorf(u1)), 0), n - 2);
  f0 = __fsub_rn(u0, float(i0));
  f1 = __fsub_rn(u1, float(i1));
}
__device__ __forceinline__ void axis_term(double l, int n, int& i0, double& f) {
  const double u = mul_rn(mul_rn(add_rn(l, 1.0), 0.5), double(n - 1));
  const double fl = floor(u);
  const int i = (fl >= 0.0 && fl <= double(n - 2)) ? int(fl) : (fl > 0.0 ? n - 2 : 0);
  i0 = i;
  f = fmin(fmax(sub_rn(u, double(i)), 0.0), 1.0);
}

template <typename T>
__device__ __forceinline__ Cell cell_of(const ModelDev<T>& md, const T* __restrict__ tfm, T x0, T x1, T x2) {
  const T l0 = local_coord(x0, x1, x2, ldg(tfm + 0), ldg(tfm + 1), ldg(tfm + 2), ldg(tfm + 3));
  const T l1 = local_coord(x0, x1, x2, ldg(tfm + 4), ldg(tfm + 5), ldg(tfm + 6), ldg(tfm + 7));
  const T l2 = local_coord(x0, x1, x2, ldg(tfm + 8), ldg(tfm + 9), ldg(tfm + 10), ldg(tfm + 11));
  Cell c;
  c.inside = (fabs(l0) <= T(1)) && (fabs(l1) <= T(1)) && (fabs(l2) <= T(1));
  axis_term(l0, md.W, c.ix, c.fx);
  axis_term(l1, md.H, c.iy, c.fy);
  axis_term(l2, md.D, c.iz, c.fz);
  return c;
}

template <typename T>
__device__ __forceinline__ double lerp_first(T a, T b, double f) {
  return add_rn(static_cast<double>(a), mul_rn(f, static_cast<double>(sub_rn(b, a))));
}
__device__ __forceinline__ double lerp_d(double a, double b, double f) { return add_rn(a, mul_rn(f, sub_rn(b, a))); }

template <typename T>
__device__ __forceinline__ T to_model(double v);
template <>
__device__ __forceinline__ float to_model<float>(double v) {
  return __double2float_rn(v);
}
template <>
__device__ __forceinline__ double to_model<double>(double v) {
  return v;
}

// Trilinear features of grid m at cell c for channel ch (c.inside assumed).
template <typename T>
__device__ __forceinline__ T interp_channel(const ModelDev<T>& md, int m, const Cell& c, int ch) {
  const int C = md.C;
  const int64_t sx = C, sy = int64_t(md.W) * C, sz = int64_t(md.H) * md.W * C;
  const T* g = md.grid + ((((int64_t)m * md.D + c.iz) * md.H + c.iy) * md.W + c.ix) * C + ch;
  const double c00 = lerp_first(ldg(g), ldg(g + sx), c.fx);
  const double c10 = lerp_first(ldg(g + sy), ldg(g + sy + sx), c.fx);
  const double c01 = lerp_first(ldg(g + sz), ldg(g + sz + sx), c.fx);
  const double c11 = lerp_first(ldg(g + sz + sy), ldg(g + sz + sy + sx), c.fx);
  return to_model<T>(lerp_d(lerp_d(c00, c10, c.fy), lerp_d(c01, c11, c.fy), c.fz));
}

// Two channels at once (C == 2, float): 8-byte vector gathers.
__device__ __forceinline__ void interp_pair(const ModelDev<float>& md, int m, const Cell& c, float& o0, float& o1) {
  const int64_t sx = 1, sy = md.W, sz = int64_t(md.H) * md.W;
  const float2* g = reinterpret_cast<const float2*>(md.grid) + (((int64_t)m * md.D + c.iz) * md.H + c.iy) * md.W + c.ix;
  const float2 a000 = __ldg(g), a001 = __ldg(g + sx), a010 = __ldg(g + sy), a011 = __ldg(g + sy + sx);
  const float2 a100 = __ldg(g + sz), a101 = __ldg(g + sz + sx), a110 = __ldg(g + sz + sy),
               a111 = __ldg(g + sz + sy + sx);
  {
    const double c00 = lerp_first(a000.x, a001.x, c.fx), c10 = lerp_first(a010.x, a011.x, c.fx);
    const double c01 = lerp_first(a100.x, a101.x, c.fx), c11 = lerp_first(a110.x, a111.x, c.fx);
    o0 = __double2float_rn(lerp_d(lerp_d(c00, c10, c.fy), lerp_d(c01, c11, c.fy), c.fz));
  }
  {
    const double c00 = lerp_first(a000.y, a001.y, c.fx), c10 = lerp_first(a010.y, a011.y, c.fx);
    const double c01 = lerp_first(a100.y, a101.y, c.fx), c11 = lerp_first(a110.y, a111.y, c.fx);
    o1 = __double2float_rn(lerp_d(lerp_d(c00, c10, c.fy), lerp_d(c01, c11, c.fy), c.fz));
  }
}

// packed fp32x2 (sm_100 FADD2 / FMUL2 / FFMA2): both channels of a corner in one
// instruction, each half rounded exactly like the scalar operation
__device__ __forceinline__ float2 f2_add(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 f2_sub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 f2_mul(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 f2_fma(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 f2_lerp(float2 a, float2 b, float t) {  // a + t (b - a), per channel
  return f2_fma(make_float2(t, t), f2_sub(b, a), a);
}

// Two channels in f32 arithmetic (training fast path: lerps rounded in f32 instead of
// f64; features differ from the bit-exact encoder by <= 1 ulp).
__device__ __forceinline__ void interp_pair_f32(const float* __restrict__ grid, int W, int HW, int vbase, float fx,
                                                float fy, float fz, float& o0, float& o1) {
  const float2* g = reinterpret_cast<const float2*>(grid) + vbase;
  const float2 a000 = __ldg(g), a001 = __ldg(g + 1), a010 = __ldg(g + W), a011 = __ldg(g + W + 1);
  const float2 a100 = __ldg(g + HW), a101 = __ldg(g + HW + 1), a110 = __ldg(g + HW + W),
               a111 = __ldg(g + HW + W + 1);
  const float2 r = f2_lerp(f2_lerp(f2_lerp(a000, a001, fx), f2_lerp(a010, a011, fx), fy),
                           f2_lerp(f2_lerp(a100, a101, fx), f2_lerp(a110, a111, fx), fy), fz);
  o0 = r.x;
  o1 = r.y;
}

// the two halves of interp_pair_f32 (8 float2 corner loads; lerps), same arithmetic and order
__device__ __forceinline__ void gather_pair_f32(const float* __restrict__ grid, int W, int HW, int vbase, float2* a) {
  const float2* g = reinterpret_cast<const float2*>(grid) + vbase;
  a[0] = __ldg(g);
  a[1] = __ldg(g + 1);
  a[2] = __ldg(g + W);
  a[3] = __ldg(g + W + 1);
  a[4] = __ldg(g + HW);
  a[5] = __ldg(g + HW + 1);
  a[6] = __ldg(g + HW + W);
  a[7] = __ldg(g + HW + W + 1);
}
__device__ __forceinline__ void lerp_pair_f32(const float2* a, float fx, float fy, float fz, float& o0, float& o1) {
  const float2 r = f2_lerp(f2_lerp(f2_lerp(a[0], a[1], fx), f2_lerp(a[2], a[3], fx), fy),
                           f2_lerp(f2_lerp(a[4], a[5], fx), f2_lerp(a[6], a[7], fx), fy), fz);
  o0 = r.x;
  o1 = r.y;
}

// the two halves of interp_pairx_f32, so a caller can issue several cells' corner loads before
// the first lerp (memory-level parallelism); same arithmetic in the same order
__device__ __forceinline__ void gather_pairx_f32(const float4* __restrict__ gx, int W, int HW, int vbase, float4* b) {
  const float4* g = gx + vbase;
#ifdef APMG_ABL_NOGATHER  // timing ablation only: no corner loads (wrong results)
  const float q = __int_as_float(vbase & 0x3fffff);
  b[0] = b[1] = b[2] = b[3] = make_float4(q, q, q, q);
  (void)g;
#else
  b[0] = __ldg(g);
  b[1] = __ldg(g + W);
  b[2] = __ldg(g + HW);
  b[3] = __ldg(g + HW + W);
#endif
}
__device__ __forceinline__ void lerp_pairx_f32(const float4* b, float fx, float fy, float fz, float& o0, float& o1) {
  const float2 r = f2_lerp(f2_lerp(f2_lerp(make_float2(b[0].x, b[0].y), make_float2(b[0].z, b[0].w), fx),
                                   f2_lerp(make_float2(b[1].x, b[1].y), make_float2(b[1].z, b[1].w), fx), fy),
                           f2_lerp(f2_lerp(make_float2(b[2].x, b[2].y), make_float2(b[2].z, b[2].w), fx),
                                   f2_lerp(make_float2(b[3].x, b[3].y), make_float2(b[3].z, b[3].w), fx), fy),
                           fz);
  o0 = r.x;
  o1 = r.y;
}

// interp_pair_f32 over the x-pair copy: 4 float4 loads instead of 8 float2, same
// arithmetic in the same order (bit-identical features)
__device__ __forceinline__ void interp_pairx_f32(const float4* __restrict__ gx, int W, int HW, int vbase, float fx,
                                                 float fy, float fz, float& o0, float& o1) {
  const float4* g = gx + vbase;
#ifdef APMG_ABL_NOGATHER  // timing ablation only: no corner loads (wrong results)
  const float q = __int_as_float(vbase & 0x3fffff);
  const float4 b00 = make_float4(q, q, q, q), b01 = b00, b10 = b00, b11 = b00;
  (void)g;
#else
  const float4 b00 = __ldg(g), b01 = __ldg(g + W), b10 = __ldg(g + HW), b11 = __ldg(g + HW + W);
#endif
  const float2 r = f2_lerp(f2_lerp(f2_lerp(make_float2(b00.x, b00.y), make_float2(b00.z, b00.w), fx),
                                   f2_lerp(make_float2(b01.x, b01.y), make_float2(b01.z, b01.w), fx), fy),
                           f2_lerp(f2_lerp(make_float2(b10.x, b10.y), make_float2(b10.z, b10.w), fx),
                                   f2_lerp(make_float2(b11.x, b11.y), make_float2(b11.z, b11.w), fx), fy),
                           fz);
  o0 = r.x;
  o1 = r.y;
}

// 256-bit read-only gather (LDG.E.256; 32-byte aligned)
__device__ __forceinline__ void ldg256(const float* p, float (&r)[8]) {
  asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7])
      : "l"(p));
}

// interp_pair_f32 over the xy-quad copy: 2 256-bit loads, same arithmetic in the same order
// (bit-identical features)
__device__ __forceinline__ void interp_pairq_f32(const float* __restrict__ gq, int HW, int vbase, float fx, float fy,
                                                 float fz, float& o0, float& o1) {
  const float* g = gq + 8 * size_t(vbase);
  float a[8], b[8];
  ldg256(g, a);
  ldg256(g + 8 * size_t(HW), b);
  const float2 r = f2_lerp(f2_lerp(f2_lerp(make_float2(a[0], a[1]), make_float2(a[2], a[3]), fx),
                                   f2_lerp(make_float2(a[4], a[5]), make_float2(a[6], a[7]), fx), fy),
                           f2_lerp(f2_lerp(make_float2(b[0], b[1]), make_float2(b[2], b[3]), fx),
                                   f2_lerp(make_float2(b[4], b[5]), make_float2(b[6], b[7]), fx), fy),
                           fz);
  o0 = r.x;
  o1 = r.y;
}

// the two halves of interp_pairq_f32 (2 256-bit loads; lerps), same arithmetic and order
__device__ __forceinline__ void gather_pairq_f32(const float* __restrict__ gq, int HW, int vbase, float* a) {
  const float* g = gq + 8 * size_t(vbase);
  float (&lo)[8] = *reinterpret_cast<float(*)[8]>(a);
  float (&hi)[8] = *reinterpret_cast<float(*)[8]>(a + 8);
  ldg256(g, lo);
  ldg256(g + 8 * size_t(HW), hi);
}
__device__ __forceinline__ void lerp_pairq_f32(const float* a, float fx, float fy, float fz, float& o0, float& o1) {
  const float2 r = f2_lerp(f2_lerp(f2_lerp(make_float2(a[0], a[1]), make_float2(a[2], a[3]), fx),
                                   f2_lerp(make_float2(a[4], a[5]), make_float2(a[6], a[7]), fx), fy),
                           f2_lerp(f2_lerp(make_float2(a[8], a[9]), make_float2(a[10], a[11]), fx),
                                   f2_lerp(make_float2(a[12], a[13]), make_float2(a[14], a[15]), fx), fy),
                           fz);
  o0 = r.x;
  o1 = r.y;
}

// Encode point (x0,x1,x2) in grid m into out[0..C) (zero outside the grid).
template <typename T>
__device__ __forceinline__ void encode_grid_point(const ModelDev<T>& md, int m, T x0, T x1, T x2, T* out,
                                                  int out_stride) {
  const Cell c = cell_of(md, md.tf + 16 * m, x0, x1, x2);
  if (!c.inside) {
    for (int ch = 0; ch < md.C; ++ch) out[ch * out_stride] = T(0);
    return;
  }
  if constexpr (sizeof(T) == 4) {
    if (md.C == 2) {
      float a, b;
      interp_pair(md, m, c, a, b);
      out[0] = a;
      out[out_stride] = b;
      return;
    }
  }
  for (int ch = 0; ch < md.C; ++ch) out[ch * out_stride] = interp_channel(md, m, c, ch);
}

__device__ __forceinline__ void atomic_add2(float* addr, float a, float b) {
  atomicAdd(reinterpret_cast<float2*>(addr), make_float2(a, b));
}

// Scatter grad g[0..C) of point (x0,x1,x2) in grid m into dgrid (channel-last),
// weights (wx*wy)*wz in f64 as optim.py:129-152; contributions rounded to T.
// float, two channels: corner weights and contributions in f32 (the fractions are exact
// in f32; the reference's f64 products differ by <= 1 ulp per contribution, far inside the
// 1e-3 gradient tolerance that float atomics already impose).
__device__ __forceinline__ void scatter_pair_f32(const ModelDev<float>& md, float* __restrict__ dgrid, int m,
                                                 const Cell& c, float g0, float g1) {
  const float fx = float(c.fx), fy = float(c.fy), fz = float(c.fz);
  const float wx[2] = {1.f - fx, fx}, wy[2] = {1.f - fy, fy}, wz[2] = {1.f - fz, fz};
  const int sy = 2 * md.W, sz = 2 * md.H * md.W;
  float* base = dgrid + (size_t(((m * md.D + c.iz) * md.H + c.iy) * md.W + c.ix) << 1);
#pragma unroll
  for (int cz = 0; cz < 2; ++cz)
#pragma unroll
    for (int cy = 0; cy < 2; ++cy) {
      const float wzy = wy[cy] * wz[cz];
      float* row = base + cz * sz + cy * sy;
#pragma unroll
      for (int cx = 0; cx < 2; ++cx) {
        const float w = wx[cx] * wzy;
        atomic_add2(row + 2 * cx, g0 * w, g1 * w);
      }
    }
}

// same from a precomputed base vertex index (vertex units, channel-last C = 2)
__device__ __forceinline__ void scatter_vertex_f32(const ModelDev<float>& md, float* __restrict__ dgrid, int vbase,
                                                   float fx, float fy, float fz, float g0, float g1) {
  const float wx[2] = {1.f - fx, fx}, wy[2] = {1.f - fy, fy}, wz[2] = {1.f - fz, fz};
  if (md.grad_pairs) {
    float4* base = reinterpret_cast<float4*>(dgrid) + vbase;
#pragma unroll
    for (int cz = 0; cz < 2; ++cz)
#pragma unroll
      for (int cy = 0; cy < 2; ++cy) {
        const float wzy = wy[cy] * wz[cz], w0 = wx[0] * wzy, w1 = wx[1] * wzy;
        atomicAdd(base + cz * md.H * md.W + cy * md.W, make_float4(g0 * w0, g1 * w0, g0 * w1, g1 * w1));
      }
    return;
  }
  const int sy = 2 * md.W, sz = 2 * md.H * md.W;
  float* base = dgrid + (size_t(vbase) << 1);
#pragma unroll
  for (int cz = 0; cz < 2; ++cz)
#pragma unroll
    for (int cy = 0; cy < 2; ++cy) {
      const float wzy = wy[cy] * wz[cz];
      float* row = base + cz * sz + cy * sy;
#pragma unroll
      for (int cx = 0; cx < 2; ++cx) {
        const float w = wx[cx] * wzy;
        atomic_add2(row + 2 * cx, g0 * w, g1 * w);
      }
    }
}

// Warp-aggregated scatter: lanes whose point falls in the same cell (same base vertex)
// of this grid are grouped with __match_any_sync, their 8 corners x 2 channel
// contributions are summed with a peer tree reduction (one shuffle round per doubling, at
// most APMG_AGG_ROUNDS rounds), and the lane heading each reduced block issues the 8
// float2 REDs.  With spatially bucketed batches a warp's 32 points cover a few cells of a
// grid, so this cuts the L2 atomics several-fold; the round cap trades a few more REDs
// (L2 RED throughput has headroom) for fewer shuffles (the crossbar is the bound).
// Must be called by all 32 lanes (invalid lanes pass valid = false).
__device__ __forceinline__ void scatter_vertex_warp_agg(const ModelDev<float>& md, float* __restrict__ dgrid,
                                                       bool valid, int vbase, float fx, float fy, float fz, float g0,
                                                       float g1) {
  const int lane = threadIdx.x & 31;
  const int key = valid ? vbase : -1 - lane;
  const unsigned peers = __match_any_sync(0xffffffffu, key);
  float2 v[8];  // corner c: (channel 0, channel 1)
  {
    const float wx[2] = {1.f - fx, fx}, wy[2] = {1.f - fy, fy}, wz[2] = {1.f - fz, fz};
    const float2 g = make_float2(g0, g1);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const float w = valid ? wx[c & 1] * (wy[(c >> 1) & 1] * wz[c >> 2]) : 0.f;
      v[c] = f2_mul(g, make_float2(w, w));
    }
  }
  const int rank = __popc(peers & ((1u << lane) - 1u));  // position within the group
  int rounds = 0;
  if (__any_sync(0xffffffffu, __popc(peers) > 1)) {
    int rel = rank;
    unsigned rem = peers & (0xfffffffeu << lane);
    while (rounds < APMG_AGG_ROUNDS && __any_sync(0xffffffffu, rem != 0u)) {
      const int next = __ffs(rem);
      const int src = next ? next - 1 : lane;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float2 t = make_float2(__shfl_sync(0xffffffffu, v[c].x, src), __shfl_sync(0xffffffffu, v[c].y, src));
        if (next) v[c] = f2_add(v[c], t);
      }
      const unsigned keep = __ballot_sync(0xffffffffu, !(rel & 1));
      rem &= keep;
      rel >>= 1;
      ++rounds;
    }
  }
  // after `rounds` rounds the lanes of rank 0 mod 2^rounds hold their block's sums
  if (!valid || (rank & ((1 << rounds) - 1)) != 0) return;
  if (md.grad_pairs) {  // x-pair gradient: corners (0, cy, cz) and (1, cy, cz) in one float4 RED
    float4* base = reinterpret_cast<float4*>(dgrid) + vbase;
#pragma unroll
    for (int c = 0; c < 8; c += 2)
#ifdef APMG_ABL_NORED  // timing ablation only: no gradient REDs (wrong results)
      if (v[c].x == 1.2345e-30f && v[c + 1].y == 1.2345e-30f) base[c] = make_float4(v[c].x, v[c].y, v[c + 1].x, v[c + 1].y);
#else
      atomicAdd(base + (c >> 2) * md.H * md.W + ((c >> 1) & 1) * md.W,
                make_float4(v[c].x, v[c].y, v[c + 1].x, v[c + 1].y));
#endif
    return;
  }
  const int sy = 2 * md.W, sz = 2 * md.H * md.W;
  float* base = dgrid + (size_t(vbase) << 1);
#pragma unroll
  for (int c = 0; c < 8; ++c) atomic_add2(base + (c >> 2) * sz + ((c >> 1) & 1) * sy + 2 * (c & 1), v[c].x, v[c].y);
}

// Leader-gather variant of the aggregated scatter: instead of tree-reducing the 8 x 2 corner
// contributions (16 shuffles per round), each block leader fetches its members' five inputs
// (g0, g1, fx, fy, fz) one member per round and forms their corner contributions itself:
// 5 shuffles per member, the weights recomputed in the FMA pipe, which has headroom (the
// shuffles share the LSU data path with the shared-memory traffic and the gathers).  Lanes
// of rank r = 0 mod (CAP + 1) in their cell group lead blocks of up to CAP + 1 lanes.
#ifndef APMG_GATHER_CAP
#define APMG_GATHER_CAP 2
#endif
// weights wx[c & 1] * (wy[(c >> 1) & 1] * wz[c >> 2]) formed in packed fp32x2 (same roundings as
// the scalar products: (wy0, wy1) * wz, then (wx0, wx1) * wzy), contributions g * w
__device__ __forceinline__ void corner_terms(float2 g, float fx, float fy, float fz, float2* v, bool add) {
  const float2 wx = make_float2(1.f - fx, fx), wy = make_float2(1.f - fy, fy);
  const float wz[2] = {1.f - fz, fz};
#pragma unroll
  for (int cz = 0; cz < 2; ++cz) {
    const float2 wzy = __fmul2_rn(wy, make_float2(wz[cz], wz[cz]));  // (cy = 0, cy = 1)
#pragma unroll
    for (int cy = 0; cy < 2; ++cy) {
      const float t = cy ? wzy.y : wzy.x;
      const float2 w = __fmul2_rn(wx, make_float2(t, t));  // (cx = 0, cx = 1)
      const int c = 4 * cz + 2 * cy;
      v[c] = add ? f2_fma(g, make_float2(w.x, w.x), v[c]) : f2_mul(g, make_float2(w.x, w.x));
      v[c + 1] = add ? f2_fma(g, make_float2(w.y, w.y), v[c + 1]) : f2_mul(g, make_float2(w.y, w.y));
    }
  }
}

// deterministic mode (FX): every cell costs 16 scalar integer REDs instead of 4 float4 REDs, so
// larger leader blocks pay there (the float sums inside a block run in lane order: still
// deterministic once the batch order inside each bucket is fixed)
#ifndef APMG_FX_GATHER_CAP
#define APMG_FX_GATHER_CAP 5  // blocks of 6: 425.6 M points/s (blocks of 4 / 5 / 7 / 8: 401 / 419 / 423 / 417)
#endif
// the REDs of one aggregated cell: 8 corners x 2 channels (x-pair float4, fixed point or float2)
template <bool FX>
__device__ __forceinline__ void emit_cell_reds(const ModelDev<float>& md, float* __restrict__ dgrid, int vbase,
                                               const float2* v) {
  if constexpr (FX) {
    unsigned long long* base = md.dgrid_fx + (size_t(vbase) << 1);
    const int sy = 2 * md.W, sz = 2 * md.H * md.W;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      unsigned long long* a = base + (c >> 2) * sz + ((c >> 1) & 1) * sy + 2 * (c & 1);
      red_fx(a, v[c].x);
      red_fx(a + 1, v[c].y);
    }
    return;
  }
  if (md.grad_pairs) {
    float4* base = reinterpret_cast<float4*>(dgrid) + vbase;
#pragma unroll
    for (int c = 0; c < 8; c += 2)
#ifdef APMG_ABL_NORED  // timing ablation only: no gradient REDs (wrong results)
      if (v[c].x == 1.2345e-30f && v[c + 1].y == 1.2345e-30f) base[c] = make_float4(v[c].x, v[c].y, v[c + 1].x, v[c + 1].y);
#else
      atomicAdd(base + (c >> 2) * md.H * md.W + ((c >> 1) & 1) * md.W,
                make_float4(v[c].x, v[c].y, v[c + 1].x, v[c + 1].y));
#endif
    return;
  }
  const int sy = 2 * md.W, sz = 2 * md.H * md.W;
  float* base = dgrid + (size_t(vbase) << 1);
#pragma unroll
  for (int c = 0; c < 8; ++c) atomic_add2(base + (c >> 2) * sz + ((c >> 1) & 1) * sy + 2 * (c & 1), v[c].x, v[c].y);
}

template <bool FX = false, int CAP = (FX ? APMG_FX_GATHER_CAP : APMG_GATHER_CAP)>  // FX: fixed-point gradient
__device__ __forceinline__ void scatter_vertex_warp_gather(const ModelDev<float>& md, float* __restrict__ dgrid,
                                                          bool valid, int vbase, float fx, float fy, float fz,
                                                          float g0, float g1) {
  const int lane = threadIdx.x & 31;
  const int key = valid ? vbase : -1 - lane;
  const unsigned peers = __match_any_sync(0xffffffffu, key);
  const int rank = __popc(peers & ((1u << lane) - 1u));
  const bool leader = valid && (rank % (CAP + 1)) == 0;
  float2 v[8];
  // members of a leader: the next CAP set bits of peers above it, fetched one per round in
  // straight-line code (no vote loop), so the compiler can interleave the shuffles and corner
  // terms of consecutive pairs; a round without a member adds zeros
  {
    unsigned above = peers & (0xfffffffeu << lane);
    corner_terms(make_float2(g0, g1), fx, fy, fz, v, false);
#pragma unroll
    for (int k = 0; k < CAP; ++k) {
      const bool has = leader && above != 0u;
      const int src = has ? __ffs(above) - 1 : lane;
      above &= above - 1u;
      const float h0 = __shfl_sync(0xffffffffu, g0, src), h1 = __shfl_sync(0xffffffffu, g1, src);
      const float ex = __shfl_sync(0xffffffffu, fx, src), ey = __shfl_sync(0xffffffffu, fy, src),
                  ez = __shfl_sync(0xffffffffu, fz, src);
      corner_terms(has ? make_float2(h0, h1) : make_float2(0.f, 0.f), ex, ey, ez, v, true);
    }
  }
  if (!leader) return;
  emit_cell_reds<FX>(md, dgrid, vbase, v);
}



template <typename T>
__device__ __forceinline__ void scatter_grid_point(const ModelDev<T>& md, T* __restrict__ dgrid, int m, T x0, T x1,
                                                   T x2, const T* g, int g_stride) {
  const Cell c = cell_of(md, md.tf + 16 * m, x0, x1, x2);
  if (!c.inside) return;
  const int C = md.C;
  if (md.dgrid_fx) {  // deterministic mode: each contribution rounded to T, then fixed point
    const int64_t fsy = int64_t(md.W) * C, fsz = int64_t(md.H) * md.W * C;
    unsigned long long* fb = md.dgrid_fx + ((((int64_t)m * md.D + c.iz) * md.H + c.iy) * md.W + c.ix) * C;
    for (int cz = 0; cz < 2; ++cz)
      for (int cy = 0; cy < 2; ++cy)
        for (int cx = 0; cx < 2; ++cx) {
          const double w = mul_rn(mul_rn(cx ? c.fx : 1.0 - c.fx, cy ? c.fy : 1.0 - c.fy), cz ? c.fz : 1.0 - c.fz);
          for (int ch = 0; ch < C; ++ch)
            red_fx(fb + cz * fsz + cy * fsy + cx * C + ch,
                   static_cast<double>(to_model<T>(mul_rn(static_cast<double>(g[ch * g_stride]), w))));
        }
    return;
  }
  if constexpr (sizeof(T) == 4) {
    if (C == 2) {
      scatter_pair_f32(md, dgrid, m, c, g[0], g[g_stride]);
      return;
    }
  }
  const int64_t sx = C, sy = int64_t(md.W) * C, sz = int64_t(md.H) * md.W * C;
  T* base = dgrid + ((((int64_t)m * md.D + c.iz) * md.H + c.iy) * md.W + c.ix) * C;
  double gv[8];
  const int nc = C < 8 ? C : 8;
  for (int ch = 0; ch < nc; ++ch) gv[ch] = static_cast<double>(g[ch * g_stride]);
#pragma unroll
  for (int cz = 0; cz < 2; ++cz) {
    const double wz = cz ? c.fz : 1.0 - c.fz;
#pragma unroll
    for (int cy = 0; cy < 2; ++cy) {
      const double wy = cy ? c.fy : 1.0 - c.fy;
#pragma unroll
      for (int cx = 0; cx < 2; ++cx) {
        const double wx = cx ? c.fx : 1.0 - c.fx;
        const double w = mul_rn(mul_rn(wx, wy), wz);
        T* dst = base + cz * sz + cy * sy + cx * sx;
        if constexpr (sizeof(T) == 4) {
          if (C == 2) {
            atomic_add2(dst, __double2float_rn(mul_rn(gv[0], w)), __double2float_rn(mul_rn(gv[1], w)));
            continue;
          }
        }
        for (int ch = 0; ch < C; ++ch) {
          const double gc = ch < 8 ? gv[ch] : static_cast<double>(g[ch * g_stride]);
          atomicAdd(dst + ch, to_model<T>(mul_rn(gc, w)));
        }
      }
    }
  }
}

}  // namespace apmg
