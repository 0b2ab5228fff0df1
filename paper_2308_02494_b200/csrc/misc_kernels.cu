// Philox batch generation, fp64 volume sampling, synthetic volumes, spatial
// hash, masked Adam and hash-dispatched decomposed inference.
#include <vector>

#include "kernels.cuh"
#include "philox.cuh"

namespace apmg {

// ---- Philox uniform (trainer.py:189 -> numpy Generator.uniform)
__global__ void k_philox_uniform(uint64_t k0, uint64_t k1, uint64_t off, int64_t count, double lo, double range,
                                 double* __restrict__ out) {
  // one thread per 4-word Philox block
  const uint64_t first_blk = off >> 2;
  const uint64_t last_blk = (off + count - 1) >> 2;
  for (uint64_t b = first_blk + blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; b <= last_blk;
       b += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t w[4];
    philox_block(b + 1, k0, k1, w);
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const uint64_t j = 4 * b + l;
      if (j >= off && j < off + uint64_t(count)) out[j - off] = add_rn(lo, mul_rn(range, word_to_double(w[l])));
    }
  }
}

// ---- fp64 trilinear volume sampling (volume.py:168-199)
struct VolAxis {
  int i0;
  double f;
  int step;
};

__device__ __forceinline__ VolAxis vol_axis(double p, int n) {
  VolAxis a;
  if (n == 1) {
    a.i0 = 0;
    a.f = 0.0;
    a.step = 0;
    return a;
  }
  const double u = mul_rn(mul_rn(add_rn(p, 1.0), 0.5), double(n - 1));
  const double fl = floor(u);
  const int i = fl < 0.0 ? 0 : (fl > double(n - 2) ? n - 2 : int(fl));
  a.i0 = i;
  a.f = sub_rn(u, double(i));
  a.step = 1;
  return a;
}

__device__ __forceinline__ double sample_trilinear(const float* __restrict__ data, int w, int h, int d, double p0,
                                                   double p1, double p2) {
  const VolAxis ax = vol_axis(p0, w), ay = vol_axis(p1, h), az = vol_axis(p2, d);
  const int64_t sx = ax.step, sy = int64_t(ay.step) * w, sz = int64_t(az.step) * w * h;
  const float* b = data + (int64_t(az.i0) * h + ay.i0) * w + ax.i0;
  const double c000 = __ldg(b), c001 = __ldg(b + sx), c010 = __ldg(b + sy), c011 = __ldg(b + sy + sx);
  const double c100 = __ldg(b + sz), c101 = __ldg(b + sz + sx), c110 = __ldg(b + sz + sy),
               c111 = __ldg(b + sz + sy + sx);
  const double x00 = lerp_d(c000, c001, ax.f), x10 = lerp_d(c010, c011, ax.f);
  const double x01 = lerp_d(c100, c101, ax.f), x11 = lerp_d(c110, c111, ax.f);
  return lerp_d(lerp_d(x00, x10, ay.f), lerp_d(x01, x11, ay.f), az.f);
}

__global__ void k_sample_volume(const float* __restrict__ data, int w, int h, int d, const double* __restrict__ pts,
                                int64_t n, double* __restrict__ out, int32_t* oob) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const double p0 = pts[3 * i], p1 = pts[3 * i + 1], p2 = pts[3 * i + 2];
    if (!(fabs(p0) <= 1.0 && fabs(p1) <= 1.0 && fabs(p2) <= 1.0)) {
      if (oob) *oob = 1;
      out[i] = 0.0;
      continue;
    }
    out[i] = sample_trilinear(data, w, h, d, p0, p1, p2);
  }
}

// ---- training batch: Philox coords (f64) -> fp64 targets -> float32 coords (trainer.py:189-191)
template <typename T>
__global__ void k_train_batch(uint64_t k0, uint64_t k1, int64_t batch, const float* __restrict__ vol, int w, int h,
                              int d, T* __restrict__ coords, T* __restrict__ targets, const TrainCtl* ctl) {
  if (ctl->skip) return;
  const uint64_t base = 3ull * uint64_t(batch) * uint64_t(ctl->it);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < batch; i += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t j = base + 3ull * uint64_t(i);
    const uint64_t b0 = j >> 2, b1 = (j + 2) >> 2;
    uint64_t wa[4], wb[4];
    philox_block(b0 + 1, k0, k1, wa);
    if (b1 != b0) philox_block(b1 + 1, k0, k1, wb);
    double c[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const uint64_t jj = j + a;
      const uint64_t word = ((jj >> 2) == b0) ? wa[jj & 3] : wb[jj & 3];
      c[a] = add_rn(-1.0, mul_rn(2.0, word_to_double(word)));
    }
    const double t = sample_trilinear(vol, w, h, d, c[0], c[1], c[2]);
    targets[i] = T(__double2float_rn(t));  // volume.sample_many(...).astype(np.float32)
    coords[3 * i] = T(__double2float_rn(c[0]));
    coords[3 * i + 1] = T(__double2float_rn(c[1]));
    coords[3 * i + 2] = T(__double2float_rn(c[2]));
  }
}

template __global__ void k_train_batch<float>(uint64_t, uint64_t, int64_t, const float*, int, int, int, float*, float*,
                                              const TrainCtl*);
template __global__ void k_train_batch<double>(uint64_t, uint64_t, int64_t, const float*, int, int, int, double*,
                                               double*, const TrainCtl*);

// ---- spatial bucketing of the batch (order-free: the losses and gradients are sums over
// points, so a permutation changes nothing but the summation order).  Points are binned
// into the Morton-ordered cells of a 32^3 lattice over [-1,1]^3 so that a 64-point tile of
// the recon kernel covers a compact region: its corner gathers hit L1 and its grid
// scatters land on a handful of cells.
__device__ __forceinline__ uint32_t spread3(uint32_t v) {
  v &= 0x3ff;
  v = (v | (v << 16)) & 0x030000FF;
  v = (v | (v << 8)) & 0x0300F00F;
  v = (v | (v << 4)) & 0x030C30C3;
  v = (v | (v << 2)) & 0x09249249;
  return v;
}

__device__ __forceinline__ uint32_t bucket_of(float x, float y, float z) {
  const int bx = min(31, max(0, int((x + 1.0f) * 16.0f)));
  const int by = min(31, max(0, int((y + 1.0f) * 16.0f)));
  const int bz = min(31, max(0, int((z + 1.0f) * 16.0f)));
  return spread3(bx) | (spread3(by) << 1) | (spread3(bz) << 2);
}

// Batch generation for the sorted path, split so that the volume is sampled in bucket
// order (coherent reads) instead of Philox order (one random DRAM sector per corner):
//   k_batch_keys      Philox coords (f64, trainer.py:189) + bucket key + bucket counts
//   k_bucket_scan     exclusive scan of the counts
//   k_bucket_scatter  f64 coords to their bucket slot
//   k_sample_sorted   fp64 trilinear targets (volume.py:147-199) + float32 coords, in place
// Targets are sampled at the f64 coordinates exactly as in k_train_batch.
__global__ void k_batch_keys(uint64_t k0, uint64_t k1, int64_t batch, double* __restrict__ c64,
                             uint32_t* __restrict__ key, int32_t* __restrict__ counts, const TrainCtl* ctl) {
  if (ctl->skip) return;
  const uint64_t base = 3ull * uint64_t(batch) * uint64_t(ctl->it);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < batch; i += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t j = base + 3ull * uint64_t(i);
    const uint64_t b0 = j >> 2, b1 = (j + 2) >> 2;
    uint64_t wa[4], wb[4];
    philox_block(b0 + 1, k0, k1, wa);
    if (b1 != b0) philox_block(b1 + 1, k0, k1, wb);
    double c[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const uint64_t jj = j + a;
      const uint64_t word = ((jj >> 2) == b0) ? wa[jj & 3] : wb[jj & 3];
      c[a] = add_rn(-1.0, mul_rn(2.0, word_to_double(word)));
      c64[3 * i + a] = c[a];
    }
    const uint32_t k = bucket_of(__double2float_rn(c[0]), __double2float_rn(c[1]), __double2float_rn(c[2]));
    key[i] = k;
    atomicAdd(&counts[k], 1);
  }
}

// in-place exclusive scan of kBuckets counts: one block of 1024 threads, 32 consecutive
// counts per thread (vector loads), warp shuffles + one smem pass across warps
constexpr int kBuckets = 32768;
__global__ void __launch_bounds__(1024) k_bucket_scan(int32_t* __restrict__ counts, const TrainCtl* ctl, int ahead) {
  if (ahead ? ctl->gen_skip : ctl->skip) return;
  __shared__ int32_t wsum[32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  int4* c4 = reinterpret_cast<int4*>(counts) + 8 * t;
  int4 v[8];
  int32_t s = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    v[q] = c4[q];
    s += v[q].x + v[q].y + v[q].z + v[q].w;
  }
  int32_t inc = s;  // inclusive scan of the per-thread sums within the warp
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, inc, off);
    if (lane >= off) inc += y;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    int32_t w = wsum[lane], wi = w;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, wi, off);
      if (lane >= off) wi += y;
    }
    wsum[lane] = wi - w;  // exclusive prefix of the warp totals
  }
  __syncthreads();
  int32_t run = wsum[warp] + inc - s;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    int4 o;
    o.x = run;
    run += v[q].x;
    o.y = run;
    run += v[q].y;
    o.z = run;
    run += v[q].z;
    o.w = run;
    run += v[q].w;
    c4[q] = o;
  }
}

__global__ void k_bucket_scatter(const double* __restrict__ c64, const uint32_t* __restrict__ key, int64_t n,
                                 int32_t* __restrict__ cursor, double* __restrict__ c64_out,
                                 int32_t* __restrict__ perm, const TrainCtl* ctl) {
  if (ctl->skip) return;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t pos = atomicAdd(&cursor[key[i]], 1);
    c64_out[3 * pos] = c64[3 * i];
    c64_out[3 * pos + 1] = c64[3 * i + 1];
    c64_out[3 * pos + 2] = c64[3 * i + 2];
    if (perm) perm[pos] = int32_t(i);
  }
}

// Deterministic mode: the atomic cursor leaves the points of a bucket in arrival order; put them
// back in batch order (one warp per bucket: rank = number of the bucket's points with a smaller
// batch index), writing c64_out.  `end` holds each bucket's end offset after the scatter.
__global__ void k_bucket_stable(const double* __restrict__ c64_in, const int32_t* __restrict__ perm,
                                const int32_t* __restrict__ end, int nbuckets, double* __restrict__ c64_out,
                                const TrainCtl* ctl) {
  if (ctl->skip) return;
  const int lane = threadIdx.x & 31;
  for (int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < nbuckets; b += (gridDim.x * blockDim.x) >> 5) {
    const int lo = b ? end[b - 1] : 0, n = end[b] - lo;
    for (int k0 = 0; k0 < n; k0 += 32) {  // warp-uniform loops: every lane reaches the shuffles
      const int k = k0 + lane;
      const int pk = k < n ? perm[lo + k] : 0x7fffffff;
      int rank = 0;
      for (int j0 = 0; j0 < n; j0 += 32) {
        const int pj = j0 + lane < n ? perm[lo + j0 + lane] : 0x7fffffff;
#pragma unroll 8
        for (int t = 0; t < 32; ++t) rank += __shfl_sync(0xffffffffu, pj, t) < pk;
      }
      if (k < n) {
        const int64_t src = lo + k, dst = lo + rank;
        c64_out[3 * dst] = c64_in[3 * src];
        c64_out[3 * dst + 1] = c64_in[3 * src + 1];
        c64_out[3 * dst + 2] = c64_in[3 * src + 2];
      }
    }
  }
}

template <typename T>
__global__ void k_sample_sorted(const double* __restrict__ c64, int64_t n, const float* __restrict__ vol, int w,
                                int h, int d, T* __restrict__ coords, T* __restrict__ targets, const TrainCtl* ctl) {
  if (ctl->skip) return;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const double c0 = c64[3 * i], c1 = c64[3 * i + 1], c2 = c64[3 * i + 2];
    targets[i] = T(__double2float_rn(sample_trilinear(vol, w, h, d, c0, c1, c2)));
    coords[3 * i] = T(__double2float_rn(c0));
    coords[3 * i + 1] = T(__double2float_rn(c1));
    coords[3 * i + 2] = T(__double2float_rn(c2));
  }
}

// ---- 8x8x8-bricked copy of the training volume: a trilinear footprint (2x2x2 voxels)
// falls in one 2 KB brick for (7/8)^3 of the points, so the sorted sampler touches ~2 DRAM
// granules per point instead of ~6 with [D][H][W] rows (values and arithmetic unchanged)
__device__ __forceinline__ int64_t brick_off(int x, int y, int z, int nbx, int nby) {
  return ((int64_t(z >> 3) * nby + (y >> 3)) * nbx + (x >> 3)) * 512 + ((z & 7) << 6) + ((y & 7) << 3) + (x & 7);
}

__global__ void k_brick_volume(const float* __restrict__ vol, int w, int h, int d, int nbx, int nby,
                               float* __restrict__ out) {
  const int64_t n = int64_t(w) * h * d;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const int x = int(i % w);
    const int64_t r = i / w;
    const int y = int(r % h), z = int(r / h);
    out[brick_off(x, y, z, nbx, nby)] = vol[i];
  }
}

template <typename T>
__global__ void k_sample_sorted_bricked(const double* __restrict__ c64, int64_t n, const float* __restrict__ bricks,
                                        int w, int h, int d, int nbx, int nby, T* __restrict__ coords,
                                        T* __restrict__ targets, const TrainCtl* ctl) {
  if (ctl->skip) return;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const double c0 = c64[3 * i], c1 = c64[3 * i + 1], c2 = c64[3 * i + 2];
    const VolAxis ax = vol_axis(c0, w), ay = vol_axis(c1, h), az = vol_axis(c2, d);
    const int x0 = ax.i0, x1 = ax.i0 + ax.step, y0 = ay.i0, y1 = ay.i0 + ay.step, z0 = az.i0, z1 = az.i0 + az.step;
    const double c000 = __ldg(bricks + brick_off(x0, y0, z0, nbx, nby));
    const double c001 = __ldg(bricks + brick_off(x1, y0, z0, nbx, nby));
    const double c010 = __ldg(bricks + brick_off(x0, y1, z0, nbx, nby));
    const double c011 = __ldg(bricks + brick_off(x1, y1, z0, nbx, nby));
    const double c100 = __ldg(bricks + brick_off(x0, y0, z1, nbx, nby));
    const double c101 = __ldg(bricks + brick_off(x1, y0, z1, nbx, nby));
    const double c110 = __ldg(bricks + brick_off(x0, y1, z1, nbx, nby));
    const double c111 = __ldg(bricks + brick_off(x1, y1, z1, nbx, nby));
    const double x00 = lerp_d(c000, c001, ax.f), x10 = lerp_d(c010, c011, ax.f);
    const double x01 = lerp_d(c100, c101, ax.f), x11 = lerp_d(c110, c111, ax.f);
    targets[i] = T(__double2float_rn(lerp_d(lerp_d(x00, x10, ay.f), lerp_d(x01, x11, ay.f), az.f)));
    coords[3 * i] = T(__double2float_rn(c0));
    coords[3 * i + 1] = T(__double2float_rn(c1));
    coords[3 * i + 2] = T(__double2float_rn(c2));
  }
}

// ---- corner-replicated copy of the training volume: the 8 trilinear corners of every cell
// contiguous (32 B, one DRAM sector per sample instead of ~4 granules), 8x the volume's bytes
__global__ void k_cell_volume(const float* __restrict__ vol, int w, int h, int d, float4* __restrict__ out) {
  const int cw = w > 1 ? w - 1 : 1, chh = h > 1 ? h - 1 : 1, cd = d > 1 ? d - 1 : 1;
  const int sx = w > 1 ? 1 : 0;
  const int64_t dy = h > 1 ? int64_t(w) : 0, dz = d > 1 ? int64_t(w) * h : 0;
  const int64_t n = int64_t(cw) * chh * cd;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const int cx = int(i % cw);
    const int64_t r = i / cw;
    const int cy = int(r % chh), cz = int(r / chh);
    const float* b = vol + (int64_t(cz) * h + cy) * w + cx;
    out[2 * i] = make_float4(b[0], b[sx], b[dy], b[dy + sx]);
    out[2 * i + 1] = make_float4(b[dz], b[dz + sx], b[dz + dy], b[dz + dy + sx]);
  }
}

template <typename T>
__global__ void k_sample_sorted_cells(const double* __restrict__ c64, int64_t n, const float4* __restrict__ cells,
                                      int w, int h, int d, T* __restrict__ coords, T* __restrict__ targets,
                                      const TrainCtl* ctl) {
  if (ctl->skip) return;
  const int cw = w > 1 ? w - 1 : 1, chh = h > 1 ? h - 1 : 1;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const double c0 = c64[3 * i], c1 = c64[3 * i + 1], c2 = c64[3 * i + 2];
    const VolAxis ax = vol_axis(c0, w), ay = vol_axis(c1, h), az = vol_axis(c2, d);
    const int64_t cell = (int64_t(az.i0) * chh + ay.i0) * cw + ax.i0;
    const float4 lo = __ldg(cells + 2 * cell), hi = __ldg(cells + 2 * cell + 1);
    const double x00 = lerp_d(double(lo.x), double(lo.y), ax.f), x10 = lerp_d(double(lo.z), double(lo.w), ax.f);
    const double x01 = lerp_d(double(hi.x), double(hi.y), ax.f), x11 = lerp_d(double(hi.z), double(hi.w), ax.f);
    targets[i] = T(__double2float_rn(lerp_d(lerp_d(x00, x10, ay.f), lerp_d(x01, x11, ay.f), az.f)));
    coords[3 * i] = T(__double2float_rn(c0));
    coords[3 * i + 1] = T(__double2float_rn(c1));
    coords[3 * i + 2] = T(__double2float_rn(c2));
  }
}

// Float sessions with the corner-replicated volume: the fp64 target is sampled while the batch is
// generated (one 32-byte cell record per point, so the Philox order costs the same DRAM sectors as
// bucket order) and the bucket scatter moves 16-byte (x, y, z, target) records straight into the
// recon kernel's coordinate / target arrays: no f64 coordinate round trip, no separate sampling
// pass.  Same values as k_batch_keys + k_bucket_scatter + k_sample_sorted_cells.
__global__ void k_batch_keys_cells(uint64_t k0, uint64_t k1, int64_t batch, const float4* __restrict__ cells, int w,
                                   int h, int d, float4* __restrict__ rec, uint32_t* __restrict__ key,
                                   int32_t* __restrict__ counts, const TrainCtl* ctl, int ahead) {
  if (ahead ? ctl->gen_skip : ctl->skip) return;
  const uint64_t base = 3ull * uint64_t(batch) * uint64_t(ahead ? ctl->gen_it : ctl->it);
  const int cw = w > 1 ? w - 1 : 1, chh = h > 1 ? h - 1 : 1;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < batch; i += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t j = base + 3ull * uint64_t(i);
    const uint64_t b0 = j >> 2, b1 = (j + 2) >> 2;
    uint64_t wa[4], wb[4];
    philox_block(b0 + 1, k0, k1, wa);
    if (b1 != b0) philox_block(b1 + 1, k0, k1, wb);
    double c[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const uint64_t jj = j + a;
      const uint64_t word = ((jj >> 2) == b0) ? wa[jj & 3] : wb[jj & 3];
      c[a] = add_rn(-1.0, mul_rn(2.0, word_to_double(word)));
    }
    const VolAxis ax = vol_axis(c[0], w), ay = vol_axis(c[1], h), az = vol_axis(c[2], d);
    const int64_t cell = (int64_t(az.i0) * chh + ay.i0) * cw + ax.i0;
    const float4 lo = __ldg(cells + 2 * cell), hi = __ldg(cells + 2 * cell + 1);
    const double x00 = lerp_d(double(lo.x), double(lo.y), ax.f), x10 = lerp_d(double(lo.z), double(lo.w), ax.f);
    const double x01 = lerp_d(double(hi.x), double(hi.y), ax.f), x11 = lerp_d(double(hi.z), double(hi.w), ax.f);
    const float x = __double2float_rn(c[0]), y = __double2float_rn(c[1]), z = __double2float_rn(c[2]);
    rec[i] = make_float4(x, y, z, __double2float_rn(lerp_d(lerp_d(x00, x10, ay.f), lerp_d(x01, x11, ay.f), az.f)));
    const uint32_t k = bucket_of(x, y, z);
    key[i] = k;
    atomicAdd(&counts[k], 1);
  }
}

// perm != nullptr (deterministic mode): the records go to the (tA, tB) halves with their batch
// index, for k_bucket_stable_rec to put each bucket back in batch order
__global__ void k_bucket_scatter_rec(const float4* __restrict__ rec, const uint32_t* __restrict__ key, int64_t n,
                                     int32_t* __restrict__ cursor, float* __restrict__ coords,
                                     float* __restrict__ targets, const TrainCtl* ctl, int ahead,
                                     float2* __restrict__ tA, float2* __restrict__ tB, int32_t* __restrict__ perm) {
  if (ahead ? ctl->gen_skip : ctl->skip) return;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t pos = atomicAdd(&cursor[key[i]], 1);
    const float4 r = rec[i];
    if (perm) {
      tA[pos] = make_float2(r.x, r.y);
      tB[pos] = make_float2(r.z, r.w);
      perm[pos] = int32_t(i);
      continue;
    }
    coords[3 * pos] = r.x;
    coords[3 * pos + 1] = r.y;
    coords[3 * pos + 2] = r.z;
    targets[pos] = r.w;
  }
}

// k_bucket_stable for the fused records: each bucket's (tA, tB) records in batch order into the
// recon inputs (one warp per bucket; rank = number of the bucket's points with a smaller index)
__global__ void k_bucket_stable_rec(const float2* __restrict__ tA, const float2* __restrict__ tB,
                                    const int32_t* __restrict__ perm, const int32_t* __restrict__ end, int nbuckets,
                                    float* __restrict__ coords, float* __restrict__ targets, const TrainCtl* ctl,
                                    int ahead) {
  if (ahead ? ctl->gen_skip : ctl->skip) return;
  const int lane = threadIdx.x & 31;
  for (int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < nbuckets; b += (gridDim.x * blockDim.x) >> 5) {
    const int lo = b ? end[b - 1] : 0, n = end[b] - lo;
    for (int k0 = 0; k0 < n; k0 += 32) {  // warp-uniform loops: every lane reaches the shuffles
      const int k = k0 + lane;
      const int pk = k < n ? perm[lo + k] : 0x7fffffff;
      int rank = 0;
      for (int j0 = 0; j0 < n; j0 += 32) {
        const int pj = j0 + lane < n ? perm[lo + j0 + lane] : 0x7fffffff;
#pragma unroll 8
        for (int t = 0; t < 32; ++t) rank += __shfl_sync(0xffffffffu, pj, t) < pk;
      }
      if (k < n) {
        const int64_t src = lo + k, dst = lo + rank;
        const float2 a = tA[src], c = tB[src];
        coords[3 * dst] = a.x;
        coords[3 * dst + 1] = a.y;
        coords[3 * dst + 2] = c.x;
        targets[dst] = c.y;
      }
    }
  }
}

template __global__ void k_sample_sorted_cells<float>(const double*, int64_t, const float4*, int, int, int, float*,
                                                      float*, const TrainCtl*);
template __global__ void k_sample_sorted_cells<double>(const double*, int64_t, const float4*, int, int, int, double*,
                                                       double*, const TrainCtl*);
template __global__ void k_sample_sorted_bricked<float>(const double*, int64_t, const float*, int, int, int, int, int,
                                                        float*, float*, const TrainCtl*);
template __global__ void k_sample_sorted_bricked<double>(const double*, int64_t, const float*, int, int, int, int,
                                                         int, double*, double*, const TrainCtl*);
template __global__ void k_sample_sorted<float>(const double*, int64_t, const float*, int, int, int, float*, float*,
                                                const TrainCtl*);
template __global__ void k_sample_sorted<double>(const double*, int64_t, const float*, int, int, int, double*, double*,
                                                 const TrainCtl*);

// ---- synth_volume (volume.py:283-296)
__global__ void k_synth(int w, int h, int d, int nb, const double* __restrict__ ex, const double* __restrict__ ey,
                        const double* __restrict__ ez, const double* __restrict__ amp, double bg, uint64_t k0,
                        uint64_t k1, double noise, float* __restrict__ out) {
  const int64_t total = int64_t(w) * h * d;
  for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < total; v += int64_t(gridDim.x) * blockDim.x) {
    const int x = int(v % w);
    const int64_t r = v / w;
    const int y = int(r % h);
    const int z = int(r / h);
    double acc = bg;
    for (int b = 0; b < nb; ++b)
      acc = add_rn(acc, mul_rn(mul_rn(mul_rn(amp[b], ez[int64_t(b) * d + z]), ey[int64_t(b) * h + y]),
                               ex[int64_t(b) * w + x]));
    if (noise > 0.0) {
      uint64_t wd[4];
      philox_block((uint64_t(v) >> 2) + 1, k0, k1, wd);
      acc = add_rn(acc, add_rn(-noise, mul_rn(add_rn(noise, noise), word_to_double(wd[v & 3]))));
    }
    out[v] = __double2float_rn(acc);
  }
}

// ---- spatial hash (decomposition.py:112-123)
template <typename P>
__device__ __forceinline__ int64_t brick_owner(P x0, P x1, P x2, int bi, int bj, int bk, bool& bad) {
  const double p[3] = {double(x0), double(x1), double(x2)};
  const int cnt[3] = {bi, bj, bk};
  int64_t cell[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (!(fabs(p[a]) <= 1.0)) bad = true;
    const double u = mul_rn(mul_rn(double(cnt[a]), add_rn(p[a], 1.0)), 0.5);
    int64_t c = int64_t(floor(u));
    if (c > cnt[a] - 1) c = cnt[a] - 1;
    if (c < 0) c = 0;
    cell[a] = c;
  }
  return cell[0] + int64_t(bi) * cell[1] + int64_t(bi) * bj * cell[2];
}

template <typename P>
__global__ void k_hash(const P* __restrict__ pts, int64_t n, int bi, int bj, int bk, int64_t* __restrict__ owner,
                       int32_t* oob) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    bool bad = false;
    owner[i] = brick_owner(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], bi, bj, bk, bad);
    if (bad && oob) *oob = 1;
  }
}

// owner + per-brick histogram (smem privatised) for decomposed inference
__global__ void k_hash_count(const float* __restrict__ pts, int64_t n, int bi, int bj, int bk,
                             int32_t* __restrict__ owner, int32_t* __restrict__ counts, int32_t* oob) {
  extern __shared__ int32_t s_cnt[];
  const int B = bi * bj * bk;
  for (int b = threadIdx.x; b < B; b += blockDim.x) s_cnt[b] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    bool bad = false;
    const int o = int(brick_owner(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], bi, bj, bk, bad));
    if (bad) *oob = 1;
    owner[i] = o;
    atomicAdd(&s_cnt[o], 1);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < B; b += blockDim.x)
    if (s_cnt[b]) atomicAdd(&counts[b], s_cnt[b]);
}

__global__ void k_bucket(const int32_t* __restrict__ owner, int64_t n, const int32_t* __restrict__ offsets,
                         int32_t* __restrict__ cursor, int32_t* __restrict__ index) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const int o = owner[i];
    const int slot = atomicAdd(&cursor[o], 1);
    index[offsets[o] + slot] = int32_t(i);
  }
}

// ---- masked Adam (optim.py:47-73)
template <typename T>
__device__ __forceinline__ void adam_elem(T& p, T g, T& m, T& v, T lr, T c1, T c2) {
  if (g == T(0)) return;
  m = add_rn(mul_rn(T(0.9), m), mul_rn(T(1.0 - 0.9), g));
  v = add_rn(mul_rn(T(0.99), v), mul_rn(T(1.0 - 0.99), mul_rn(g, g)));
  p = sub_rn(p, div_rn(mul_rn(lr, div_rn(m, c1)), add_rn(sqrt_rn(div_rn(v, c2)), T(1e-8))));
}

template <typename T>
__global__ void k_adam(T* __restrict__ p, const T* __restrict__ g, T* __restrict__ m, T* __restrict__ v, int64_t n,
                       double lr, double bc1, double bc2) {
  const T lr_t = T(lr), c1 = T(bc1), c2 = T(bc2);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    T pi = p[i], mi = m[i], vi = v[i];
    const T gi = g[i];
    if (gi == T(0)) continue;
    adam_elem(pi, gi, mi, vi, lr_t, c1, c2);
    p[i] = pi;
    m[i] = mi;
    v[i] = vi;
  }
}

// training variant: scalars from the controller; consumes and clears the gradient
// training variant: also keeps the x-pair grid copy (ModelDev::gridx) current: element e
// of the two-channel grid (cell e/2, channel e%2) is the low half of gridx[cell] and the
// high half of gridx[cell - 1].  gx = nullptr: no copy.
// dgx != nullptr: the grid part of the gradient is in the x-pair layout (ModelDev::grad_pairs);
// element (cell c, channel ch) sums dgx[c].lo and dgx[c - 1].hi, and clears both.
template <typename T>
__global__ void k_adam_train(T* __restrict__ p, T* __restrict__ g, T* __restrict__ m, T* __restrict__ v, int64_t n,
                             const TrainCtl* ctl, float* __restrict__ gx, int64_t gx_elems, int qw,
                             float* __restrict__ dgx, unsigned long long* __restrict__ gfx, int64_t fx_elems) {
  if (ctl->skip) return;
  const T lr_t = T(ctl->lr_main_t), c1 = T(ctl->bc1_main), c2 = T(ctl->bc2_main);
  int64_t i0 = 0;
  if constexpr (sizeof(T) == 4) {
    if (dgx && gx && !gfx) {
      // x-pair grid cells, one two-channel cell per thread and step (8-byte accesses):
      // grad(grid[c]) = dgx[c].lo + dgx[c - 1].hi, each half consumed (and cleared) by exactly
      // one cell's thread; the packed copy gets gx[c].lo = gx[c - 1].hi = grid[c]
      const int64_t cells = gx_elems >> 1;
      float2* p2 = reinterpret_cast<float2*>(p);
      float2* m2 = reinterpret_cast<float2*>(m);
      float2* v2 = reinterpret_cast<float2*>(v);
      float2* d2 = reinterpret_cast<float2*>(dgx);
      float2* x2 = reinterpret_cast<float2*>(gx);
      for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < cells;
           c += int64_t(gridDim.x) * blockDim.x) {
        const float2 lo = d2[2 * c], hi = c > 0 ? d2[2 * c - 1] : make_float2(0.f, 0.f);
        const float g0 = lo.x + hi.x, g1 = lo.y + hi.y;
        // clear both halves first: non-zero halves that cancel exactly still have to go
        if (lo.x != 0.f || lo.y != 0.f) d2[2 * c] = make_float2(0.f, 0.f);
        if (hi.x != 0.f || hi.y != 0.f) d2[2 * c - 1] = make_float2(0.f, 0.f);
        if (g0 == 0.f && g1 == 0.f) continue;
        float2 pc = p2[c], mc = m2[c], vc = v2[c];
        adam_elem(pc.x, g0, mc.x, vc.x, lr_t, c1, c2);
        adam_elem(pc.y, g1, mc.y, vc.y, lr_t, c1, c2);
        p2[c] = pc;
        m2[c] = mc;
        v2[c] = vc;
        if (qw) {  // xy-quad copy: cell c is slot 0 of quad c, 1 of c - 1, 2 of c - W, 3 of c - W - 1
          x2[4 * c] = pc;
          if (c >= 1) x2[4 * (c - 1) + 1] = pc;
          if (c >= qw) x2[4 * (c - qw) + 2] = pc;
          if (c >= qw + 1) x2[4 * (c - qw - 1) + 3] = pc;
        } else {
          x2[2 * c] = pc;
          if (c > 0) x2[2 * c - 1] = pc;
        }
      }
      i0 = 2 * cells;
    }
  }
  for (int64_t i = i0 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const bool pair = sizeof(T) == 4 && dgx && i < gx_elems;
    const bool fx = gfx && i < fx_elems;  // deterministic mode: fixed-point grid gradient
    T gi = (pair || fx) ? T(0) : g[i];
    if (fx) {
      const unsigned long long q = gfx[i];
      if (q) {
        gfx[i] = 0ull;
        gi = T(double(static_cast<long long>(q)) * kFxInv);
      }
    }
    if constexpr (sizeof(T) == 4) {
      if (pair) {
        const int64_t c = i >> 1, ch = i & 1;
        const float lo = dgx[4 * c + ch], hi = c > 0 ? dgx[4 * (c - 1) + 2 + ch] : 0.f;
        if (lo != 0.f) dgx[4 * c + ch] = 0.f;
        if (hi != 0.f) dgx[4 * (c - 1) + 2 + ch] = 0.f;
        gi = lo + hi;
      }
    }
    if (gi == T(0)) continue;
    T pi = p[i], mi = m[i], vi = v[i];
    adam_elem(pi, gi, mi, vi, lr_t, c1, c2);
    p[i] = pi;
    m[i] = mi;
    v[i] = vi;
    if (!pair && !fx) g[i] = T(0);
    if constexpr (sizeof(T) == 4) {
      if (gx && i < gx_elems) {
        const int64_t c = i >> 1, ch = i & 1;
        if (qw) {
          gx[8 * c + ch] = pi;
          if (c >= 1) gx[8 * (c - 1) + 2 + ch] = pi;
          if (c >= qw) gx[8 * (c - qw) + 4 + ch] = pi;
          if (c >= qw + 1) gx[8 * (c - qw - 1) + 6 + ch] = pi;
        } else {
          gx[4 * c + ch] = pi;
          if (c > 0) gx[4 * (c - 1) + 2 + ch] = pi;
        }
      }
    }
  }
}

template __global__ void k_adam_train<float>(float*, float*, float*, float*, int64_t, const TrainCtl*, float*,
                                             int64_t, int, float*, unsigned long long*, int64_t);
template __global__ void k_adam_train<double>(double*, double*, double*, double*, int64_t, const TrainCtl*, float*,
                                              int64_t, int, float*, unsigned long long*, int64_t);

// gridx[c] = (grid[c], grid[c + 1]) for the flat two-channel cells c (zero past the end)
__global__ void k_pack_gridx(const float2* __restrict__ grid, float4* __restrict__ gx, int64_t cells) {
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < cells; c += int64_t(gridDim.x) * blockDim.x) {
    const float2 a = grid[c], b = c + 1 < cells ? grid[c + 1] : make_float2(0.f, 0.f);
    gx[c] = make_float4(a.x, a.y, b.x, b.y);
  }
}

// xy-quad copy: gq[c] = (grid[c], grid[c + 1], grid[c + W], grid[c + W + 1]) (zero past the end)
__global__ void k_pack_gridq(const float2* __restrict__ grid, float4* __restrict__ gq, int64_t cells, int W) {
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < cells; c += int64_t(gridDim.x) * blockDim.x) {
    const float2 z = make_float2(0.f, 0.f);
    const float2 a = grid[c], b = c + 1 < cells ? grid[c + 1] : z, d = c + W < cells ? grid[c + W] : z,
                 e = c + W + 1 < cells ? grid[c + W + 1] : z;
    gq[2 * c] = make_float4(a.x, a.y, b.x, b.y);
    gq[2 * c + 1] = make_float4(d.x, d.y, e.x, e.y);
  }
}

int elementwise_grid(int64_t n, int per_sm) {
  return int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), int64_t(num_sms()) * per_sm)));
}

}  // namespace apmg

using namespace apmg;

extern "C" int apmg_philox_uniform(uint64_t key0, uint64_t key1, uint64_t word_offset, int64_t count, double lo,
                                   double hi, double* out, void* stream) {
  if (count <= 0) return APMG_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t blocks = ((word_offset + count - 1) >> 2) - (word_offset >> 2) + 1;
  APMG_LAUNCH("philox_uniform", k_philox_uniform, elementwise_grid(blocks, 8), 256, 0, st, key0, key1, word_offset,
              count, lo, hi - lo, out);
  return APMG_OK;
}

extern "C" int apmg_sample_volume(const float* data, int32_t w, int32_t h, int32_t d, const double* pts, int64_t n,
                                  double* out, int32_t* oob, void* stream) {
  APMG_ARG_CHECK(w >= 1 && h >= 1 && d >= 1, "volume dims must be positive");
  if (n <= 0) return APMG_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  APMG_LAUNCH("sample_volume", k_sample_volume, elementwise_grid(n, 8), 256, 0, st, data, w, h, d, pts, n, out, oob);
  return APMG_OK;
}

extern "C" int apmg_synth_volume(int32_t w, int32_t h, int32_t d, int32_t nblobs, const double* ex, const double* ey,
                                 const double* ez, const double* amp, double background, uint64_t key0, uint64_t key1,
                                 double noise, float* out, void* stream) {
  APMG_ARG_CHECK(w >= 1 && h >= 1 && d >= 1, "dims must be positive");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t total = int64_t(w) * h * d;
  APMG_LAUNCH("synth_volume", k_synth, elementwise_grid(total, 16), 256, 0, st, w, h, d, nblobs, ex, ey, ez, amp,
              background, key0, key1, noise, out);
  return APMG_OK;
}

extern "C" int apmg_spatial_hash(int32_t pts_dtype, const void* pts, int64_t n, int32_t bi, int32_t bj, int32_t bk,
                                 int64_t* owner, int32_t* oob, void* stream) {
  APMG_ARG_CHECK(bi >= 1 && bj >= 1 && bk >= 1, "brick counts must be >= 1");
  if (n <= 0) return APMG_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (pts_dtype == APMG_F32)
    APMG_LAUNCH("spatial_hash", k_hash<float>, elementwise_grid(n, 8), 256, 0, st, static_cast<const float*>(pts), n,
                bi, bj, bk, owner, oob);
  else
    APMG_LAUNCH("spatial_hash", k_hash<double>, elementwise_grid(n, 8), 256, 0, st, static_cast<const double*>(pts),
                n, bi, bj, bk, owner, oob);
  return APMG_OK;
}

// ---- query routing across ranks (decomposition.py:294-304 DecomposedField.forward over ranks):
// owner-rank histogram (shared-memory privatised), host prefix sum, counting-sort scatter of the
// point indices; rows permuted to / from that order by one gather kernel
__global__ void k_owner_count(const int64_t* __restrict__ dest, int64_t n, int world, int32_t* __restrict__ counts,
                              int32_t* bad) {
  extern __shared__ int32_t s_cnt[];
  for (int b = threadIdx.x; b < world; b += blockDim.x) s_cnt[b] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t o = dest[i];
    if (o < 0 || o >= world) {
      *bad = 1;
      continue;
    }
    atomicAdd(&s_cnt[o], 1);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < world; b += blockDim.x)
    if (s_cnt[b]) atomicAdd(&counts[b], s_cnt[b]);
}

__global__ void k_owner_bucket(const int64_t* __restrict__ dest, int64_t n, const int32_t* __restrict__ offsets,
                               int32_t* __restrict__ cursor, int64_t* __restrict__ perm) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t o = dest[i];
    perm[offsets[o] + atomicAdd(&cursor[o], 1)] = i;
  }
}

// dst[r] = src[perm[r]] (gather) or dst[perm[r]] = src[r] (scatter), rows of `cols` 4-byte words
__global__ void k_permute_rows(const uint32_t* __restrict__ src, const int64_t* __restrict__ perm, int64_t n,
                               int cols, int scatter, uint32_t* __restrict__ dst) {
  const int64_t total = n * cols;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = e / cols, c = e - r * cols, q = perm[r];
    if (scatter)
      dst[q * cols + c] = src[e];
    else
      dst[e] = src[q * cols + c];
  }
}

extern "C" size_t apmg_owner_bucket_workspace_bytes(int32_t world) {
  Carver c(nullptr, 0);
  c.take<int32_t>(3 * size_t(world > 0 ? world : 1) + 1);
  return c.used + 256;
}

extern "C" int apmg_owner_bucket(const int64_t* dest, int64_t n, int32_t world, int64_t* perm, int64_t* counts,
                                 void* workspace, size_t workspace_bytes, void* stream) {
  APMG_ARG_CHECK(world >= 1 && world <= 4096, "world size must be in [1, 4096]");
  APMG_ARG_CHECK(counts != nullptr, "null counts");
  for (int r = 0; r < world; ++r) counts[r] = 0;
  if (n <= 0) return APMG_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Carver c(workspace, workspace_bytes);
  int32_t* d_counts = c.take<int32_t>(3 * size_t(world) + 1);  // counts | offsets | cursors | flag
  int32_t* d_off = d_counts + world;
  int32_t* d_cur = d_off + world;
  int32_t* bad = d_cur + world;
  if (!c.ok()) {
    set_error("owner bucket workspace too small");
    return APMG_E_WORKSPACE;
  }
  APMG_CUDA_TRY(cudaMemsetAsync(d_counts, 0, sizeof(int32_t) * (3 * size_t(world) + 1), st));
  APMG_LAUNCH("owner_count", k_owner_count, elementwise_grid(n, 8), 256, sizeof(int32_t) * world, st, dest, n, world,
              d_counts, bad);
  std::vector<int32_t> h(world + 1), off(world);
  APMG_CUDA_TRY(cudaMemcpyAsync(h.data(), d_counts, sizeof(int32_t) * world, cudaMemcpyDeviceToHost, st));
  APMG_CUDA_TRY(cudaMemcpyAsync(&h[world], bad, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  APMG_CUDA_TRY(cudaStreamSynchronize(st));
  APMG_ARG_CHECK(!h[world], "owner rank outside [0, world)");
  int32_t run = 0;
  for (int r = 0; r < world; ++r) {
    off[r] = run;
    run += h[r];
    counts[r] = h[r];
  }
  APMG_CUDA_TRY(cudaMemcpyAsync(d_off, off.data(), sizeof(int32_t) * world, cudaMemcpyHostToDevice, st));
  APMG_LAUNCH("owner_bucket", k_owner_bucket, elementwise_grid(n, 8), 256, 0, st, dest, n, d_off, d_cur, perm);
  APMG_CUDA_TRY(cudaStreamSynchronize(st));  // the host offsets must outlive the copy
  return APMG_OK;
}

extern "C" int apmg_permute_rows(const void* src, const int64_t* perm, int64_t n, int32_t row_words, int32_t scatter,
                                 void* dst, void* stream) {
  APMG_ARG_CHECK(row_words >= 1, "row width must be >= 1 word");
  if (n <= 0) return APMG_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  APMG_LAUNCH("permute_rows", k_permute_rows, elementwise_grid(n * row_words, 8), 256, 0, st,
              static_cast<const uint32_t*>(src), perm, n, row_words, scatter, static_cast<uint32_t*>(dst));
  return APMG_OK;
}

extern "C" int apmg_adam_step(int32_t dtype, void* params, const void* grads, void* m, void* v, int64_t n, double lr,
                              double bc1, double bc2, void* stream) {
  if (n <= 0) return APMG_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == APMG_F32)
    APMG_LAUNCH("adam", k_adam<float>, elementwise_grid(n, 8), 256, 0, st, static_cast<float*>(params),
                static_cast<const float*>(grads), static_cast<float*>(m), static_cast<float*>(v), n, lr, bc1, bc2);
  else
    APMG_LAUNCH("adam", k_adam<double>, elementwise_grid(n, 8), 256, 0, st, static_cast<double*>(params),
                static_cast<const double*>(grads), static_cast<double*>(m), static_cast<double*>(v), n, lr, bc1, bc2);
  return APMG_OK;
}

extern "C" size_t apmg_decomposed_workspace_bytes(int32_t bricks, int64_t n) {
  Carver c(nullptr, 0);
  c.take<int32_t>(n);           // owner
  c.take<int32_t>(n);           // index
  c.take<int32_t>(bricks);      // counts
  c.take<int32_t>(bricks);      // offsets
  c.take<int32_t>(bricks);      // cursor
  c.take<int32_t>(1);           // oob
  return c.used + 256;
}

static int decomposed_forward(const apmg_model* models, int32_t bricks, int32_t bi, int32_t bj, int32_t bk,
                              const double* scale, const double* offset, const float* pts, int64_t n, float* out,
                              void* workspace, size_t workspace_bytes, void* stream, int tc) {
  APMG_ARG_CHECK(bricks == bi * bj * bk && bricks >= 1, "model count does not match brick counts");
  if (n <= 0) return APMG_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Carver c(workspace, workspace_bytes);
  int32_t* owner = c.take<int32_t>(n);
  int32_t* index = c.take<int32_t>(n);
  int32_t* counts = c.take<int32_t>(bricks);
  int32_t* offsets = c.take<int32_t>(bricks);
  int32_t* cursor = c.take<int32_t>(bricks);
  int32_t* oob = c.take<int32_t>(1);
  if (!c.ok()) {
    set_error("decomposed workspace too small");
    return APMG_E_WORKSPACE;
  }
  APMG_CUDA_TRY(cudaMemsetAsync(counts, 0, sizeof(int32_t) * bricks, st));
  APMG_CUDA_TRY(cudaMemsetAsync(cursor, 0, sizeof(int32_t) * bricks, st));
  APMG_CUDA_TRY(cudaMemsetAsync(oob, 0, sizeof(int32_t), st));
  APMG_LAUNCH("hash_count", k_hash_count, elementwise_grid(n, 8), 256, sizeof(int32_t) * bricks, st, pts, n, bi, bj,
              bk, owner, counts, oob);
  std::vector<int32_t> h_counts(bricks + 1), h_off(bricks);
  APMG_CUDA_TRY(cudaMemcpyAsync(h_counts.data(), counts, sizeof(int32_t) * bricks, cudaMemcpyDeviceToHost, st));
  APMG_CUDA_TRY(cudaMemcpyAsync(&h_counts[bricks], oob, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  APMG_CUDA_TRY(cudaStreamSynchronize(st));
  if (h_counts[bricks]) {
    set_error("coordinate outside [-1, 1]^3");
    return APMG_E_ARG;
  }
  int32_t run = 0;
  for (int b = 0; b < bricks; ++b) {
    h_off[b] = run;
    run += h_counts[b];
  }
  APMG_CUDA_TRY(cudaMemcpyAsync(offsets, h_off.data(), sizeof(int32_t) * bricks, cudaMemcpyHostToDevice, st));
  APMG_LAUNCH("bucket", k_bucket, elementwise_grid(n, 8), 256, 0, st, owner, n, offsets, cursor, index);
  for (int b = 0; b < bricks; ++b) {
    if (!h_counts[b]) continue;
    int rc = apmg_internal_forward_gather(&models[b], scale + 3 * b, offset + 3 * b, pts, index + h_off[b],
                                          h_counts[b], out, st, tc);
    if (rc) return rc;
  }
  // keep the host staging alive until the H2D copy has been consumed
  APMG_CUDA_TRY(cudaStreamSynchronize(st));
  return APMG_OK;
}

extern "C" int apmg_decomposed_forward(const apmg_model* models, int32_t bricks, int32_t bi, int32_t bj, int32_t bk,
                                       const double* scale, const double* offset, const float* pts, int64_t n,
                                       float* out, void* workspace, size_t workspace_bytes, void* stream) {
  return decomposed_forward(models, bricks, bi, bj, bk, scale, offset, pts, n, out, workspace, workspace_bytes, stream,
                            0);
}

extern "C" int apmg_decomposed_forward_tc(const apmg_model* models, int32_t bricks, int32_t bi, int32_t bj,
                                          int32_t bk, const double* scale, const double* offset, const float* pts,
                                          int64_t n, float* out, void* workspace, size_t workspace_bytes,
                                          void* stream) {
  return decomposed_forward(models, bricks, bi, bj, bk, scale, offset, pts, n, out, workspace, workspace_bytes, stream,
                            1);
}
