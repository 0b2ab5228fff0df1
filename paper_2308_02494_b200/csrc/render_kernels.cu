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

// render.py:202-220 per pixel, from the host's camera basis (fwd, right, true_up, tan_half,
// aspect): the same f64 chain numpy evaluates -- u = px tan_half aspect, v = py tan_half,
// d = (fwd + u right) + v up, |d| = sqrt((d0^2 + d1^2) + d2^2), d / |d| -- so the directions are
// bit-identical to generate_rays.
struct CamBasis {
  double f[3], r[3], u[3], tan_half, aspect;
};
__global__ void k_generate_rays(CamBasis cb, int W, int H, double* __restrict__ dirs) {
  const int64_t n = int64_t(W) * H;
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < n; q += int64_t(gridDim.x) * blockDim.x) {
    const int j = int(q / W), i = int(q - int64_t(j) * W);
    const double px = __dsub_rn(__dmul_rn(__ddiv_rn(__dadd_rn(double(i), 0.5), double(W)), 2.0), 1.0);
    const double py = __dsub_rn(1.0, __dmul_rn(__ddiv_rn(__dadd_rn(double(j), 0.5), double(H)), 2.0));
    const double u = __dmul_rn(__dmul_rn(px, cb.tan_half), cb.aspect), v = __dmul_rn(py, cb.tan_half);
    double d[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) d[k] = __dadd_rn(__dadd_rn(cb.f[k], __dmul_rn(u, cb.r[k])), __dmul_rn(v, cb.u[k]));
    const double nrm = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(d[0], d[0]), __dmul_rn(d[1], d[1])),
                                            __dmul_rn(d[2], d[2])));
#pragma unroll
    for (int k = 0; k < 3; ++k) dirs[3 * q + k] = __ddiv_rn(d[k], nrm);
  }
}

// render.py:286-290 for rays ray_ids[0..nr), samples s0 .. s0+cs-1 of S: dt = (exit - enter) / S,
// sample s at t = (s + 0.5) dt + enter, p = clip(origin + t dir, -1, 1) -> float32
__global__ void k_ray_points(RayOrigin org, const double* __restrict__ dirs, const int64_t* __restrict__ ray_ids,
                             int64_t nr, int32_t S, int32_t s0, int32_t cs, const double* __restrict__ enter,
                             const double* __restrict__ exit_t, float* __restrict__ pts) {
  const int64_t total = nr * cs;
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < total; q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = q / cs;
    const int s = s0 + int(q - j * cs);
    const int64_t r = ray_ids[j];
    const double* d = dirs + 3 * r;
    const double e = enter[r];
    const double dt = __ddiv_rn(__dsub_rn(exit_t[r], e), double(S));
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

// One chunk of samples (s0 .. s0+cs-1 of S) of rays ray_ids: field values [nr][cs] ->
// transfer function -> front-to-back update of the per-ray state (r, g, b, alpha), indexed by
// ray id.  Chunked marching lets the host drop rays that reached the early-exit opacity before
// their remaining samples are queried: the reference evaluates them and discards the result,
// so the pixels are the same.
__global__ void k_composite_chunk(const float* __restrict__ values, const int64_t* __restrict__ ray_ids, int64_t nr,
                                  int32_t S, int32_t cs, const double* __restrict__ enter,
                                  const double* __restrict__ exit_t, const float4* __restrict__ lut, TfParams tp,
                                  CompParams cp, float4* __restrict__ state) {
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < nr; j += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = ray_ids[j];
    const float step = __double2float_rn(__ddiv_rn(__dsub_rn(exit_t[r], enter[r]), double(S)));
    const float e = __fdiv_rn(step, cp.ref_step);
    float4 st = state[r];
    const float* v = values + j * cs;
    for (int s = 0; s < cs; ++s) {
      if (cp.early_on && !(st.w < cp.early)) break;
      const float4 c = tf_apply(lut, tp, v[s]);
      const float corr = __fsub_rn(1.f, powf(__fsub_rn(1.f, c.w), e));
      const float contrib = __fmul_rn(__fsub_rn(1.f, st.w), corr);
      st.x = __fadd_rn(st.x, __fmul_rn(contrib, c.x));
      st.y = __fadd_rn(st.y, __fmul_rn(contrib, c.y));
      st.z = __fadd_rn(st.z, __fmul_rn(contrib, c.z));
      st.w = __fadd_rn(st.w, contrib);
    }
    state[r] = st;
  }
}

// background blend of the final state of rays ray_ids (render.py:258-263)
__global__ void k_composite_finish(const int64_t* __restrict__ ray_ids, int64_t nr, const float4* __restrict__ state,
                                   CompParams cp, float4* __restrict__ out) {
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < nr; j += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = ray_ids[j];
    const float4 st = state[r];
    const float rem = __fmul_rn(__fsub_rn(1.f, st.w), cp.bg[3]);
    out[r] = make_float4(__fadd_rn(st.x, __fmul_rn(rem, cp.bg[0])), __fadd_rn(st.y, __fmul_rn(rem, cp.bg[1])),
                         __fadd_rn(st.z, __fmul_rn(rem, cp.bg[2])), __fadd_rn(st.w, rem));
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

extern "C" int apmg_generate_rays(const double* basis, int32_t width, int32_t height, double* dirs, void* stream) {
  APMG_ARG_CHECK(basis && width >= 1 && height >= 1 && dirs, "bad camera arguments");
  CamBasis cb{{basis[0], basis[1], basis[2]}, {basis[3], basis[4], basis[5]}, {basis[6], basis[7], basis[8]},
              basis[9], basis[10]};
  const int64_t n = int64_t(width) * height;
  APMG_LAUNCH("generate_rays", k_generate_rays, elementwise_grid(n, 8), 256, 0, static_cast<cudaStream_t>(stream),
              cb, width, height, dirs);
  return APMG_OK;
}

extern "C" int apmg_ray_points(const double* origin, const double* dirs, const int64_t* ray_ids, int64_t nr,
                               int32_t samples, int32_t s0, int32_t count, const double* enter, const double* exit_t,
                               float* pts, void* stream) {
  APMG_ARG_CHECK(origin && samples >= 1 && s0 >= 0 && count >= 0 && s0 + count <= samples, "bad sample range");
  if (nr == 0 || count == 0) return APMG_OK;
  APMG_ARG_CHECK(dirs && ray_ids && enter && exit_t && pts, "null argument");
  APMG_LAUNCH("ray_points", k_ray_points, elementwise_grid(nr * count, 8), 256, 0,
              static_cast<cudaStream_t>(stream), origin_of(origin), dirs, ray_ids, nr, samples, s0, count, enter,
              exit_t, pts);
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

extern "C" int apmg_composite_chunk(const float* values, const int64_t* ray_ids, int64_t nr, int32_t samples,
                                    int32_t count, const double* enter, const double* exit_t, const float* lut,
                                    const float* tf, const float* comp, float* state, void* stream) {
  APMG_ARG_CHECK(tf && comp && samples >= 1 && count >= 0, "null parameters or bad sample counts");
  if (nr == 0 || count == 0) return APMG_OK;
  APMG_ARG_CHECK(values && ray_ids && enter && exit_t && lut && state, "null argument");
  APMG_LAUNCH("composite", k_composite_chunk, elementwise_grid(nr, 4), 128, 0, static_cast<cudaStream_t>(stream),
              values, ray_ids, nr, samples, count, enter, exit_t, reinterpret_cast<const float4*>(lut),
              tf_params(tf), comp_params(comp), reinterpret_cast<float4*>(state));
  return APMG_OK;
}

extern "C" int apmg_composite_finish(const int64_t* ray_ids, int64_t nr, const float* state, const float* comp,
                                     float* out, void* stream) {
  APMG_ARG_CHECK(comp, "null parameters");
  if (nr == 0) return APMG_OK;
  APMG_ARG_CHECK(ray_ids && state && out, "null argument");
  APMG_LAUNCH("composite_finish", k_composite_finish, elementwise_grid(nr, 4), 128, 0,
              static_cast<cudaStream_t>(stream), ray_ids, nr, reinterpret_cast<const float4*>(state),
              comp_params(comp), reinterpret_cast<float4*>(out));
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
