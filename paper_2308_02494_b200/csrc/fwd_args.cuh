// Arguments and point sources of the forward sweeps (SIMT k_forward and the tensor-core
// lattice kernel k_infer_tc).  Reference: model.py:164-166, trainer.py:226-247,
// decomposition.py:294-304.
#pragma once

#include "kernels.cuh"

namespace apmg {

// Point sources for the forward tile kernel.
enum FwdMode : int { kFwdPts = 0, kFwdFeats = 1, kFwdLattice = 2, kFwdGather = 3 };

template <typename T>
struct FwdArgs {
  ModelDev<T> md;
  int mode;
  int64_t n;
  const T* pts;         // kFwdPts: [n][3]
  const T* feats;       // kFwdFeats: [n][F]
  T* out;               // kFwdPts / kFwdFeats: [n]
  // lattice sweep (kFwdLattice): voxel box of a (W,H,D) lattice
  int LW, LH, LD, bx0, by0, bz0, bw, bh;
  int affine;
  int stamps;           // k_infer_tc phase stamps (profiling aid)
  int box_local;        // truth / recon are dense [bd][bh][bw] arrays of the box (brick sweeps)
  int tc_points;        // kFwdPts through the tensor-core sweep kernel (f32 lerps, bf16x3 MLP)
  double sc0, sc1, sc2, of0, of1, of2;
  const float* truth;   // [LD][LH][LW] or null
  float* recon;         // [LD][LH][LW] or null
  double* sse;          // accumulated when truth != null: sse_part[block] per CTA, then k_sse_finalize
  double* sse_part;     // [gridDim.x] per-CTA sums (fixed-order final reduction: deterministic)
  // gather (kFwdGather): global f32 points through an index list
  const float* gpts;    // [*][3]
  const int32_t* index; // [n] point ids of this brick
  float* gout;          // out[index[i]]
};

// truth / recon element of box voxel (x, y, z): global lattice index, or box-local
template <typename T>
__device__ __forceinline__ int64_t lattice_elem(const FwdArgs<T>& a, int x, int y, int z) {
  if (a.box_local) return (int64_t(z) * a.bh + y) * a.bw + x;
  return (int64_t(a.bz0 + z) * a.LH + (a.by0 + y)) * a.LW + (a.bx0 + x);
}

// f64 lattice coordinate of vertex i of n (axis_coords, volume.py:161-165)
__device__ __forceinline__ double lattice_coord(int i, int n) {
  if (n == 1) return 0.0;
  return sub_rn(div_rn(mul_rn(2.0, double(i)), double(n - 1)), 1.0);
}

template <typename T>
__device__ __forceinline__ void fwd_point(const FwdArgs<T>& a, int64_t i, T& x0, T& x1, T& x2) {
  if (a.mode == kFwdPts) {
    x0 = a.pts[3 * i];
    x1 = a.pts[3 * i + 1];
    x2 = a.pts[3 * i + 2];
    return;
  }
  double g0, g1, g2;
  if (a.mode == kFwdLattice) {
    const int64_t plane = int64_t(a.bw) * a.bh;
    const int z = int(i / plane);
    const int64_t r = i - z * plane;
    const int y = int(r / a.bw);
    const int x = int(r - int64_t(y) * a.bw);
    // psnr casts the f64 lattice coordinates to float32 before predicting (trainer.py:240)
    g0 = double(__double2float_rn(lattice_coord(a.bx0 + x, a.LW)));
    g1 = double(__double2float_rn(lattice_coord(a.by0 + y, a.LH)));
    g2 = double(__double2float_rn(lattice_coord(a.bz0 + z, a.LD)));
  } else {  // kFwdGather
    const int64_t id = a.index[i];
    g0 = a.gpts[3 * id];
    g1 = a.gpts[3 * id + 1];
    g2 = a.gpts[3 * id + 2];
  }
  if (a.affine) {  // DecomposedField: f64 brick affine then float32 (decomposition.py:302-303)
    g0 = add_rn(mul_rn(g0, a.sc0), a.of0);
    g1 = add_rn(mul_rn(g1, a.sc1), a.of1);
    g2 = add_rn(mul_rn(g2, a.sc2), a.of2);
  }
  x0 = T(__double2float_rn(g0));
  x1 = T(__double2float_rn(g1));
  x2 = T(__double2float_rn(g2));
}


// tensor-core lattice sweep for the flagship shape (infer_tc.cu)
bool infer_tc_eligible(const FwdArgs<float>& a);
int launch_infer_tc(const FwdArgs<float>& a, cudaStream_t st);

}  // namespace apmg
