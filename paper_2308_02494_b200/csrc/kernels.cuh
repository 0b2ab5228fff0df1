// Internal declarations shared by the kernel translation units.
#pragma once

#include <algorithm>

#include "common.cuh"
#include "mlp_tile.cuh"
#include "model_dev.cuh"

namespace apmg {

// Device-resident state of the training loop (trainer.py:170-220).  Written by
// the single-warp controller kernels only; every other kernel reads `skip`
// (the loop has ended) and `density_on` (this iteration runs a density step).
struct TrainCtl {
  int32_t skip;
  int32_t finished;
  int32_t transforms_active;
  int32_t density_on;
  int64_t it;              // index of the iteration being executed
  int64_t iterations_run;
  int64_t t_main, t_tf;    // Adam step counters of the two groups (trainer.py:178-179)
  int64_t stop_iteration;  // -1 until the transform stop rule fires
  int64_t n_triggers;
  int64_t dens_count;      // length of density_history
  int64_t plat_count;      // length of PlateauState.history since the last clear
  double lr_scale;
  double l_rec, l_dens;
  double lr_main_t, bc1_main, bc2_main;  // this iteration's Adam scalars (main group)
  double lr_tf_t, bc1_tf, bc2_tf;        // this iteration's Adam scalars (transform group)
  // batch generated one iteration ahead on the session's side stream (float sessions with the
  // corner-replicated volume): its iteration index and skip flag, written by ctl_begin
  int64_t gen_it;
  int32_t gen_skip;
  int32_t pad_;
};

template <typename T>
int launch_recon(const ModelDev<T>& md, int64_t n, const T* coords, const T* targets, T* sq, double* loss, T* dgrid,
                 T* dw1, T* dw2, T* dw3, void* ws, size_t wsb, const TrainCtl* ctl, double* l_rec_log,
                 cudaStream_t st);
template <typename T>
size_t recon_ws_bytes(int F, int64_t n);

bool recon_tc_eligible(const ModelDev<float>& md);
// launch_recon<float> on this model shape runs the bf16x3 tcgen05 kernel (recon_tc16.cu)
bool recon_uses_tc16(const apmg_model& m);
// grid for grid-stride elementwise kernels: enough 256-thread blocks for n, at most per_sm per SM
int elementwise_grid(int64_t n, int per_sm);
// fixed-order sum of the per-CTA SSE partials of a lattice sweep into *sse (model_kernels.cu)
int launch_sse_finalize(const double* part, int n, double* sse, cudaStream_t st);
// gridx[c] = (grid[c], grid[c + 1]) over the flat two-channel cells (misc_kernels.cu)
__global__ void k_pack_gridx(const float2* __restrict__ grid, float4* __restrict__ gx, int64_t cells);
// xy-quad copy (ModelDev::gridq): two float4 per cell (misc_kernels.cu)
__global__ void k_pack_gridq(const float2* __restrict__ grid, float4* __restrict__ gq, int64_t cells, int W);
int launch_recon_tc16(const ModelDev<float>& md, int64_t n, const float* coords, const float* targets, float* sq,
                      float* dgrid, float* part_dw, double* part_loss, int grid, const TrainCtl* ctl, cudaStream_t st);

template <typename T, typename TE>
int launch_density(T* tf, int M, int p, const T* x, const TE* err, int64_t n, double* loss, T* dtf, double* rho_total,
                   T* adam_m, T* adam_v, void* ws, size_t wsb, const TrainCtl* ctl, cudaStream_t st,
                   int pre_nb = 0);
// the rho / partial-sum slots of launch_density's workspace, for a producer that fills them
// ahead of it (the fused recon kernel; then launch_density(..., pre_nb = its CTA count))
int density_rho_slots(int M, int64_t n, void* ws, size_t wsb, double** rho, double** part1);
// the recon tc16 kernel's CTA count for a batch of n points
int recon_tc16_grid(int64_t n);
size_t density_ws_bytes(int M, int64_t n);

}  // namespace apmg

int apmg_internal_forward_gather(const apmg_model* m, const double* sc, const double* of, const float* pts,
                                 const int32_t* index, int64_t n, float* out, cudaStream_t st, int tc = 0);
