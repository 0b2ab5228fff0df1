// Renderer field-query path: ray / box intersection, ray-march sample
// points, transfer-function lookup and front-to-back emission-absorption compositing.
//
// Reference: render.py:206-226 (ray_box_hits), :229-264 (_corrected_alpha, composite_ray,
// _composite), :126-138 (TransferFunction.apply), :274-298 (_render_rays).  The field values
// between the point and composite passes come from the library's own field kernels (model
// forward, decomposed forward, fp64 volume sampling).
//
// Numerics follow the reference's elementwise chains: f64 ray geometry with separate mul /
// add roundings (numpy never fuses), f32 transfer function and compositing written with
// explicit _rn intrinsics so nvcc cannot contract them into FMAs.  The one libm difference is
// powf (CUDA: <= 2 ulp; the reference's numpy float32 power: libm powf).
#include <math_constants.h>

#include "kernels.cuh"

namespace apmg {

struct RayOrigin {
  double o[3];
};

// render.py:206-226: slab test against [-1, 1]^3, NaN-propagating min / max like numpy
__device__ __forceinline__ double np_min(double a, double b) { return (a != a || b != b) ? a + b : (a < b ? a : b); }
__device__ __forceinline__ double np_max(double a, double b) { return (a != a || b != b) ? a + b : (a > b ? a : b); }

__device__ __forceinline__ void box_hit(const RayOrigin& org, const double* d, double& enter, double& exit_t,
                                        bool& hit) {
  double t0 = -CUDART_INF, t1 = CUDART_INF;
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    const double o = org.o[ax], di = d[ax];
    const double ta = __ddiv_rn(__dsub_rn(-1.0, o), di);
    const double tb = __ddiv_rn(__dsub_rn(1.0, o), di);
    const double near_t = np_min(ta, tb), far_t = np_max(ta, tb);
    if (di == 0.0) {
      const bool inside = fabs(o) <= 1.0;
      t0 = inside ? t0 : CUDART_INF;
      t1 = inside ? t1 : -CUDART_INF;
    } else {
      t0 = np_max(t0, near_t);
      t1 = np_min(t1, far_t);
    }
  }
  enter = np_max(t0, 0.0);
  exit_t = t1;
  hit = (t1 > enter) && (t1 > 0.0) && isfinite(enter);
}

__global__ void k_ray_box_hits(RayOrigin org, const double* __restrict__ dirs, int64_t n, double* __restrict__ enter,
                               double* __restrict__ exit_t, uint8_t* __restrict__ hit) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    double e, x;
    bool h;
    box_hit(org, dirs + 3 * i, e, x, h);
    enter[i] = e;
    exit_t[i] = x;
    hit[i] = h ? 1 : 0;
  }
}

// render.py:286-290 for rays ray_ids[0..nr): dt = (exit - enter) / S, sample s at
// t = (s + 0.5) dt + enter, p = clip(origin + t dir, -1, 1) -> float32
__global__ void k_ray_points(RayOrigin org, const double* __restrict__ dirs, const int64_t* __restrict__ ray_ids,
                             int64_t nr, int32_t S, float* __restrict__ pts, double* __restrict__ dt_out) {
  const int64_t total = nr * S;
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < total; q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = q / S;
    const int s = int(q - j * S);
    const double* d = dirs + 3 * ray_ids[j];
    double e, x;
    bool h;
    box_hit(org, d, e, x, h);
    const double dt = __ddiv_rn(__dsub_rn(x, e), double(S));
    if (s == 0) dt_out[j] = dt;
    const double t = __dadd_rn(__dmul_rn(__dadd_rn(double(s), 0.5), dt), e);
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      double p = __dadd_rn(org.o[ax], __dmul_rn(t, d[ax]));
      p = fmin(fmax(p, -1.0), 1.0);
      pts[3 * q + ax] = __double2float_rn(p);
    }
  }
}

struct TfParams {
  float vmin, span;  // np.float32(vmin), np.float32(vmax - vmin); span_ok = vmax > vmin
  float lo, win;     // np.float32(lo), np.float32(hi - lo)
  int span_ok;
};

// render.py:126-138 (TransferFunction.apply) for one value
__device__ __forceinline__ float4 tf_apply(const float4* __restrict__ lut, const TfParams& p, float v) {
  const float nrm = p.span_ok ? __fdiv_rn(__fsub_rn(v, p.vmin), p.span) : 0.f;
  float w = __fdiv_rn(__fsub_rn(nrm, p.lo), p.win);
  w = fminf(fmaxf(w, 0.f), 1.f);
  const float pos = __fmul_rn(w, 255.f);
  const int i0 = min(int(pos), 254);
  const float frac = __fsub_rn(pos, float(i0));
  const float4 a = lut[i0], b = lut[i0 + 1];
  const float g = __fsub_rn(1.f, frac);
  return make_float4(__fadd_rn(__fmul_rn(a.x, g), __fmul_rn(b.x, frac)),
                     __fadd_rn(__fmul_rn(a.y, g), __fmul_rn(b.y, frac)),
                     __fadd_rn(__fmul_rn(a.z, g), __fmul_rn(b.z, frac)),
                     __fadd_rn(__fmul_rn(a.w, g), __fmul_rn(b.w, frac)));
}

__global__ void k_tf_apply(const float* __restrict__ values, int64_t n, const float4* __restrict__ lut, TfParams p,
                           float4* __restrict__ out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = tf_apply(lut, p, values[i]);
}

struct CompParams {
  float ref_step;     // np.float32(reference_step)
  float bg[4];
  float early;        // early_exit_alpha (when early_on)
  int early_on;
};

// render.py:240-264 (_composite) for one ray; rgba(s) yields sample s
template <typename Sample>
__device__ __forceinline__ float4 composite(Sample rgba, int S, float step, const CompParams& c) {
  const float e = __fdiv_rn(step, c.ref_step);
  float r = 0.f, g = 0.f, b = 0.f, alpha = 0.f;
  for (int s = 0; s < S; ++s) {
    if (c.early_on && !(alpha < c.early)) break;  // inactive from here on: nothing changes
    const float4 v = rgba(s);
    const float corr = __fsub_rn(1.f, powf(__fsub_rn(1.f, v.w), e));
    const float contrib = __fmul_rn(__fsub_rn(1.f, alpha), corr);
    r = __fadd_rn(r, __fmul_rn(contrib, v.x));
    g = __fadd_rn(g, __fmul_rn(contrib, v.y));
    b = __fadd_rn(b, __fmul_rn(contrib, v.z));
    alpha = __fadd_rn(alpha, contrib);
  }
  const float rem = __fmul_rn(__fsub_rn(1.f, alpha), c.bg[3]);
  return make_float4(__fadd_rn(r, __fmul_rn(rem, c.bg[0])), __fadd_rn(g, __fmul_rn(rem, c.bg[1])),
                     __fadd_rn(b, __fmul_rn(rem, c.bg[2])), __fadd_rn(alpha, rem));
}

// field values [nr][S] of rays ray_ids -> transfer function -> composite -> out[ray_ids[j]]
__global__ void k_composite_values(const float* __restrict__ values, const double* __restrict__ dt,
                                   const int64_t* __restrict__ ray_ids, int64_t nr, int32_t S,
                                   const float4* __restrict__ lut, TfParams tp, CompParams cp,
                                   float4* __restrict__ out) {
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < nr; j += int64_t(gridDim.x) * blockDim.x) {
    const float* v = values + j * S;
    const float4 o = composite([&](int s) { return tf_apply(lut, tp, v[s]); }, S, __double2float_rn(dt[j]), cp);
    out[ray_ids ? ray_ids[j] : j] = o;
  }
}

// RGBA samples [nr][S] with per-ray steps (composite_ray / _composite)
__global__ void k_composite_rgba(const float4* __restrict__ samples, const float* __restrict__ steps, int64_t nr,
                                 int32_t S, CompParams cp, float4* __restrict__ out) {
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < nr; j += int64_t(gridDim.x) * blockDim.x) {
    const float4* v = samples + j * S;
    out[j] = composite([&](int s) { return v[s]; }, S, steps[j], cp);
  }
}

static RayOrigin origin_of(const double* o) { return RayOrigin{{o[0], o[1], o[2]}}; }
static TfParams tf_params(const float* tf) {  // [vmin, span, lo, win, span_ok]
  return TfParams{tf[0], tf[1], tf[2], tf[3], tf[4] != 0.f ? 1 : 0};
}
static CompParams comp_params(const float* c) {  // [ref_step, bg0..3, early, early_on]
  return CompParams{c[0], {c[1], c[2], c[3], c[4]}, c[5], c[6] != 0.f ? 1 : 0};
}

}  // namespace apmg

using namespace apmg;

extern "C" int apmg_ray_box_hits(const double* origin, const double* dirs, int64_t n, double* enter, double* exit_t,
                                 uint8_t* hit, void* stream) {
  APMG_ARG_CHECK(origin && (n == 0 || (dirs && enter && exit_t && hit)), "null argument");
  if (n == 0) return APMG_OK;
  APMG_LAUNCH("ray_box_hits", k_ray_box_hits, elementwise_grid(n, 8), 256, 0, static_cast<cudaStream_t>(stream),
              origin_of(origin), dirs, n, enter, exit_t, hit);
  return APMG_OK;
}

extern "C" int apmg_ray_points(const double* origin, const double* dirs, const int64_t* ray_ids, int64_t nr,
                               int32_t samples, float* pts, double* dt, void* stream) {
  APMG_ARG_CHECK(origin && samples >= 1, "null origin or samples < 1");
  if (nr == 0) return APMG_OK;
  APMG_ARG_CHECK(dirs && ray_ids && pts && dt, "null argument");
  APMG_LAUNCH("ray_points", k_ray_points, elementwise_grid(nr * samples, 8), 256, 0,
              static_cast<cudaStream_t>(stream), origin_of(origin), dirs, ray_ids, nr, samples, pts, dt);
  return APMG_OK;
}

extern "C" int apmg_tf_apply(const float* values, int64_t n, const float* lut, const float* tf, float* rgba,
                             void* stream) {
  APMG_ARG_CHECK(tf, "null transfer-function parameters");
  if (n == 0) return APMG_OK;
  APMG_ARG_CHECK(values && lut && rgba, "null argument");
  APMG_LAUNCH("tf_apply", k_tf_apply, elementwise_grid(n, 8), 256, 0, static_cast<cudaStream_t>(stream), values, n,
              reinterpret_cast<const float4*>(lut), tf_params(tf), reinterpret_cast<float4*>(rgba));
  return APMG_OK;
}

extern "C" int apmg_composite_values(const float* values, const double* dt, const int64_t* ray_ids, int64_t nr,
                                     int32_t samples, const float* lut, const float* tf, const float* comp, float* out,
                                     void* stream) {
  APMG_ARG_CHECK(tf && comp && samples >= 1, "null parameters or samples < 1");
  if (nr == 0) return APMG_OK;
  APMG_ARG_CHECK(values && dt && lut && out, "null argument");
  APMG_LAUNCH("composite", k_composite_values, elementwise_grid(nr, 4), 128, 0, static_cast<cudaStream_t>(stream),
              values, dt, ray_ids, nr, samples, reinterpret_cast<const float4*>(lut), tf_params(tf), comp_params(comp),
              reinterpret_cast<float4*>(out));
  return APMG_OK;
}

extern "C" int apmg_composite_rgba(const float* samples, const float* steps, int64_t nr, int32_t count,
                                   const float* comp, float* out, void* stream) {
  APMG_ARG_CHECK(comp && count >= 0, "null parameters");
  if (nr == 0) return APMG_OK;
  APMG_ARG_CHECK((samples || count == 0) && steps && out, "null argument");
  APMG_LAUNCH("composite_rgba", k_composite_rgba, elementwise_grid(nr, 4), 128, 0, static_cast<cudaStream_t>(stream),
              reinterpret_cast<const float4*>(samples), steps, nr, count, comp_params(comp),
              reinterpret_cast<float4*>(out));
  return APMG_OK;
}
