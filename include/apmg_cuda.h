/*
 * apmg_cuda.h -- C ABI of libapmg_cuda.so, the sm_100a implementation of the
 * APMGSRN train-and-query hot path (arXiv 2308.02494).
 *
 * The reference (/root/reference/pkg/src/apmg, pure numpy) has no FFI layer:
 * its boundary is the Python module API.  Each entry point below replaces one
 * reference function; the replaced symbol is cited as file:line relative to
 * /root/reference/pkg/src/apmg.  INTEGRATION.md shows the ctypes stub a
 * maintainer of the reference would add to bind them.
 *
 * Conventions
 *  - Every tensor argument is a DEVICE pointer unless documented otherwise;
 *    sizes are element counts.  `stream` is a cudaStream_t (NULL = legacy).
 *  - Functions return 0 on success or a negative APMG_E* code; the message is
 *    available from apmg_last_error() (thread-local).  Calls are asynchronous
 *    on `stream` unless documented as synchronising.
 *  - `dtype` is APMG_F32 or APMG_F64: the element type of the model tensors
 *    (the reference runs float32 models and float64 copies, model.py:125-136).
 *  - Device grids are CHANNEL-LAST [M][D][H][W][C]; the reference layout
 *    [M][C][D][H][W] (model.py:90) is converted by the host wrapper.
 *  - No entry point falls back to the CPU.
 */
#ifndef APMG_CUDA_H
#define APMG_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define APMG_F32 0
#define APMG_F64 1

#define APMG_OK 0
#define APMG_E_ARG (-1)        /* invalid argument / shape (ValueError in the reference) */
#define APMG_E_CUDA (-2)       /* CUDA runtime error */
#define APMG_E_WORKSPACE (-3)  /* workspace too small */
#define APMG_E_UNSUPPORTED (-4)

/* Model parameters (ApmgModel, model.py:86-119). hidden must be 64 (model.py:37). */
typedef struct apmg_model {
  int32_t dtype;
  int32_t grids, channels, depth, height, width; /* M, C, D, H, W */
  int32_t hidden;
  int32_t flat_top_p;
  const void* transforms; /* [M][4][4] */
  const void* grids_cl;   /* [M][D][H][W][C] channel-last */
  const void* w1;         /* [64][M*C] */
  const void* w2;         /* [64][64] */
  const void* w3;         /* [1][64] */
  double vmin, vmax;
} apmg_model;

/* ---- library ---------------------------------------------------------- */
const char* apmg_last_error(void);
const char* apmg_version(void);
int apmg_device_sm_count(void);
/* number of kernels this library launched since load (evidence for bench.py) */
uint64_t apmg_launch_count(void);
/* per-kernel CUDA-event timing on the launching stream (bench roofline). */
/* ---- renderer field-query path (render.py) ---------------------
 * ray_box_hits (render.py:206-226): slab test of rays (origin HOST f64[3], dirs [n][3] f64)
 * against [-1,1]^3 -> enter / exit [n] f64, hit [n] u8. */
int apmg_ray_box_hits(const double* origin, const double* dirs, int64_t n, double* enter, double* exit_t,
                      uint8_t* hit, void* stream);
/* generate_rays (render.py:202-220) on the device: basis = HOST f64[11] {fwd[3], right[3],
 * true_up[3], tan(fov/2), width/height} from the host's camera setup -> dirs [height*width][3]
 * f64, row-major from the top-left pixel, bit-identical to the numpy chain. */
int apmg_generate_rays(const double* basis, int32_t width, int32_t height, double* dirs, void* stream);
/* _render_rays sample points (render.py:286-290): samples s0 .. s0+count-1 of `samples` per ray
 * for the rays ray_ids [nr] (i64, hit rays; enter / exit [*] f64 from apmg_ray_box_hits):
 * pts [nr][count][3] f32 = clip(origin + ((s+0.5) dt + enter) dir, -1, 1), dt = (exit-enter)/samples. */
int apmg_ray_points(const double* origin, const double* dirs, const int64_t* ray_ids, int64_t nr, int32_t samples,
                    int32_t s0, int32_t count, const double* enter, const double* exit_t, float* pts,
                    void* stream);
/* TransferFunction.apply (render.py:126-138): values [n] f32 -> rgba [n][4] f32 through the
 * baked LUT [256][4] f32; tf = HOST f32[5] {vmin, vmax - vmin, lo, hi - lo, vmax > vmin}. */
int apmg_tf_apply(const float* values, int64_t n, const float* lut, const float* tf, float* rgba, void* stream);
/* _render_rays tail (render.py:292-295), one chunk of `count` samples per ray: field values
 * [nr][count] -> transfer function -> front-to-back update (render.py:240-257) of the per-ray
 * state [*][4] f32 (r, g, b, alpha; zero-initialised, indexed by ray id).  Rays whose alpha
 * reached the early-exit threshold stop accumulating.  comp = HOST f32[7] {reference_step,
 * background[4], early_exit_alpha, early_on}. */
int apmg_composite_chunk(const float* values, const int64_t* ray_ids, int64_t nr, int32_t samples, int32_t count,
                         const double* enter, const double* exit_t, const float* lut, const float* tf,
                         const float* comp, float* state, void* stream);
/* background blend of the final state (render.py:258-263) -> out[ray_ids[j]] RGBA f32. */
int apmg_composite_finish(const int64_t* ray_ids, int64_t nr, const float* state, const float* comp, float* out,
                          void* stream);
/* _composite of RGBA samples [nr][count][4] with per-ray steps [nr] f32 (composite_ray). */
int apmg_composite_rgba(const float* samples, const float* steps, int64_t nr, int32_t count, const float* comp,
                        float* out, void* stream);

/* Release the device blocks the library caches between sessions (the bricked volume
 * copy of apmg_train_create).  No reference counterpart (memory management of the CUDA
 * path). */
int apmg_release_cached(void);
/* Page-lock an existing host range in place (cudaHostRegister) so uploads from it are single DMA
 * transfers, and undo it.  Host plumbing for Volume.device_data / to_device (volume.py:225-241
 * loads the volume the reference samples in trainer.py:189); not part of the reference API. */
int apmg_host_register(void* ptr, size_t bytes);
int apmg_host_unregister(void* ptr);
/* host -> device copy on `stream` (cudaMemcpyAsync; a DMA when the host range is page-locked) */
int apmg_copy_h2d(void* dst, const void* src, size_t bytes, void* stream);
int apmg_kernel_timing_enable(int on);
/* copies up to `cap` records (name, total_ms, launches); returns count.  Synchronises. */
int apmg_kernel_timing_read(char* names /* cap*64 bytes */, double* total_ms, int64_t* launches, int cap);

/* ---- model forward (model.py:141-166) ----------------------------------- */
/* to_local (model.py:179-182): one transform [4][4], pts [n][3] -> local [n][3] (dtype) */
int apmg_to_local(int32_t dtype, const void* transform, const void* pts, int64_t n, void* out, void* stream);
/* ApmgModel.encode (model.py:141-150): pts [n][3] dtype -> feats [n][M*C] dtype */
int apmg_encode(const apmg_model* m, const void* pts, int64_t n, void* feats, void* stream);
/* ApmgModel.decode (model.py:152-162): feats [n][M*C] -> out [n] */
int apmg_decode(const apmg_model* m, const void* feats, int64_t n, void* out, void* stream);
/* ApmgModel.forward (model.py:164-166): fused encode + decode, pts [n][3] -> out [n] */
int apmg_forward(const apmg_model* m, const void* pts, int64_t n, void* out, void* stream);
/* forward of a float32 point list through the tensor-core sweep kernel (the renderer's field
 * queries): f32 lerps and bf16x3 MLP products -- within the forward gate (<= 1e-4 of the
 * value range) of model.py:164-166 but not bit-equal to apmg_forward; other model shapes
 * take apmg_forward's kernel. */
int apmg_forward_tc(const apmg_model* m, const float* pts, int64_t n, float* out, void* stream);

/* ---- reconstruction loss (optim.py:102-155) ------------------------------ */
size_t apmg_recon_workspace_bytes(const apmg_model* m, int64_t n);
/* recon_loss_and_grads: loss (device f64 scalar), sq_errors [n] dtype, and the
 * gradients of the main group: grads[0] = d grids (channel-last, ACCUMULATED:
 * must be zero on entry), grads[1..3] = d w1 [64][M*C], d w2 [64][64], d w3 [64]
 * (overwritten).  The transforms receive no gradient from this loss (optim.py:105-107). */
int apmg_recon_loss_grads(const apmg_model* m, const void* coords, const void* targets, int64_t n,
                          void* sq_errors, double* loss, void* const* grads, void* workspace,
                          size_t workspace_bytes, void* stream);

/* ---- feature density (density.py, optim.py:158-200) ---------------------- */
size_t apmg_density_workspace_bytes(int32_t grids, int64_t n);
/* density_loss_and_grads: coords [n][3] dtype, errors [n] f64 -> loss (device f64),
 * d_transforms [M][4][4] dtype (bottom rows zero).  Also writes the batch sum of
 * rho to *rho_total (device f64) so the caller can raise the reference's
 * "degenerate" DensityError (density.py:115). */
int apmg_density_loss_grads(const apmg_model* m, const void* coords, const double* errors, int64_t n,
                            double* loss, void* d_transforms, double* rho_total, void* workspace,
                            size_t workspace_bytes, void* stream);
/* feature_density (density.py:83-108): transforms [M][4][4] dtype, pts [n][3] f64 -> rho [n] f64 */
int apmg_feature_density(int32_t dtype, const void* transforms, int32_t grids, int32_t p,
                         const double* pts, int64_t n, double* rho, void* stream);
/* feature_density_terms (density.py:83-103): local [M][n][3], dets [M], bumps [M][n], rho [n] (all f64) */
int apmg_density_terms(int32_t dtype, const void* transforms, int32_t grids, int32_t p, const double* pts,
                       int64_t n, double* local, double* dets, double* bumps, double* rho, void* stream);
/* target_density (density.py:120-137) elementwise: rho_star[n] */
int apmg_target_density(const double* rho_scaled, const double* errors, int64_t n, double mean_error,
                        double eps, double* rho_star, void* stream);
/* deterministic f64 sum of x[n] (used for scale_density, means, density_loss) */
size_t apmg_sum_workspace_bytes(int64_t n);
int apmg_sum_f64(const double* x, int64_t n, double* out, void* workspace, size_t workspace_bytes,
                 void* stream);
/* density_loss (density.py:140-148) terms: out[i] = rho_s (log(rho_s+eps) - log rho*) ; caller sums/N */
int apmg_density_loss_terms(const double* rho_scaled, const double* rho_star, int64_t n, double eps,
                            double* terms, void* stream);
/* out[i] = x[i] * scale (scale_density, density.py:111-117, with scale = 1/sum) */
int apmg_scale_f64(const double* x, int64_t n, const double* divisor, double* out, void* stream);

/* ---- optimizer (optim.py:47-73) ------------------------------------------ */
/* masked Adam: entries with g == 0 leave p, m, v untouched. lr, bc1 = 1-0.9^t,
 * bc2 = 1-0.99^t are the reference's Python floats; they are rounded to dtype
 * exactly as numpy does for a float32 array operand. */
int apmg_adam_step(int32_t dtype, void* params, const void* grads, void* m, void* v, int64_t n,
                   double lr, double bc1, double bc2, void* stream);

/* ---- batch generation (trainer.py:175-191, volume.py:147-199) -------------- */
/* out[i] = lo + (hi-lo) * ((word(offset+i) >> 11) * 2^-53), word j = lane j%4 of
 * Philox4x64-10(counter = j/4 + 1, key) -- numpy.random.Philox + Generator.uniform. */
int apmg_philox_uniform(uint64_t key0, uint64_t key1, uint64_t word_offset, int64_t count, double lo,
                        double hi, double* out, void* stream);
/* Volume.sample_many: fp64 trilinear of data [D][H][W] f32 at pts [n][3] f64.
 * *oob (device int) is set to 1 if any coordinate lies outside [-1,1]^3. */
int apmg_sample_volume(const float* data, int32_t w, int32_t h, int32_t d, const double* pts, int64_t n,
                       double* out, int32_t* oob, void* stream);
/* synth_volume (volume.py:275-296): acc = background + sum_b amp_b ez[z] ey[y] ex[x]
 * (+ Philox uniform noise), rounded to f32.  ex/ey/ez are [nblobs][W|H|D] f64 device arrays. */
int apmg_synth_volume(int32_t w, int32_t h, int32_t d, int32_t nblobs, const double* ex,
                      const double* ey, const double* ez, const double* amp, double background,
                      uint64_t key0, uint64_t key1, double noise, float* out, void* stream);

/* ---- query path (decomposition.py:112-123, 294-304; trainer.py:226-247) ----- */
/* spatial_hash: pts [n][3] (dtype) -> owner [n] int64; *oob set when |p| > 1 */
int apmg_spatial_hash(int32_t pts_dtype, const void* pts, int64_t n, int32_t bi, int32_t bj, int32_t bk,
                      int64_t* owner, int32_t* oob, void* stream);
/* DecomposedField.forward: models[b] (HOST array of descriptors whose tensor
 * pointers are device pointers), per-brick affine scale/offset [B][3] (HOST f64),
 * pts [n][3] f32 -> out [n] f32.  Synchronises (reads per-brick counts). */
/* Query routing across ranks (replaces the per-owner loop of decomposition.py:294-304 when the
 * bricks live on different ranks): counting sort of n points by owner rank dest[i] in [0, world)
 * (device int64) -> perm (device int64 [n], points grouped by rank) and counts (HOST int64
 * [world]); synchronising (the counts size the all-to-all). */
size_t apmg_owner_bucket_workspace_bytes(int32_t world);
int apmg_owner_bucket(const int64_t* dest, int64_t n, int32_t world, int64_t* perm, int64_t* counts, void* workspace,
                      size_t workspace_bytes, void* stream);
/* rows of row_words 4-byte words: dst[r] = src[perm[r]] (scatter = 0) or dst[perm[r]] = src[r] */
int apmg_permute_rows(const void* src, const int64_t* perm, int64_t n, int32_t row_words, int32_t scatter, void* dst,
                      void* stream);
size_t apmg_decomposed_workspace_bytes(int32_t bricks, int64_t n);
int apmg_decomposed_forward(const apmg_model* models, int32_t bricks, int32_t bi, int32_t bj, int32_t bk,
                            const double* scale, const double* offset, const float* pts, int64_t n,
                            float* out, void* workspace, size_t workspace_bytes, void* stream);
/* apmg_decomposed_forward through the tensor-core sweep kernel per brick (the renderer's
 * decomposed-field queries): within the forward gate of the exact path, not bit-equal to it. */
int apmg_decomposed_forward_tc(const apmg_model* models, int32_t bricks, int32_t bi, int32_t bj, int32_t bk,
                               const double* scale, const double* offset, const float* pts, int64_t n, float* out,
                               void* workspace, size_t workspace_bytes, void* stream);
/* Lattice sweep of one model over the voxel box [x0,x1]x[y0,y1]x[z0,z1] of a
 * (W,H,D) lattice (axis_coords, volume.py:161-165), optionally through a
 * brick affine (scale/offset HOST f64[3] or NULL).  If truth != NULL the f64
 * sum of squared errors against truth [D][H][W] is ADDED to *sse (device f64);
 * if recon != NULL predictions are written to recon [D][H][W] f32. */
int apmg_lattice_sweep(const apmg_model* m, int32_t w, int32_t h, int32_t d, const int32_t box[6],
                       const double* scale, const double* offset, const float* truth, double* sse,
                       float* recon, void* stream);
/* Same sweep with box-local truth / recon: dense [bd][bh][bw] arrays of the box only
 * (per-rank brick inference over a volume no single GPU holds; decomposition.py:294-304
 * with trainer.py:226-247 per brick). */
int apmg_brick_sweep(const apmg_model* m, int32_t w, int32_t h, int32_t d, const int32_t box[6],
                     const double* scale, const double* offset, const float* truth_box, double* sse,
                     float* recon_box, void* stream);

/* ---- device-resident training loop (trainer.py:160-223) -------------------- */
typedef struct apmg_train_config {
  int64_t iterations, batch_size;
  double lr_main, lr_transform;
  int64_t delay_start, transform_ma_window;
  double transform_improve_threshold;
  int64_t hard_stop_iteration; /* ceil(transform_hard_stop_fraction * iterations) */
  int64_t plateau_window;
  double plateau_threshold, plateau_factor;
  int64_t plateau_max_triggers;
  uint64_t key0, key1; /* Philox key of TrainConfig.seed */
  int32_t train_transforms, plateau_enabled;
  /* 1: run-to-run bit-deterministic training (the reference's determinism contract,
   * test_acceptance.py:332-367): batch order within each spatial bucket restored by a stable
   * pass, grid gradient accumulated in 64-bit fixed point (2^-44) with integer REDs.  0: float
   * REDs in arrival order (faster; sums differ in the last bits between runs). */
  int32_t deterministic;
  int32_t reserved; /* bit 0: plain launches, no CUDA graph (sessions driven concurrently from
                     * several host threads: a capture must not overlap other threads' CUDA calls) */
} apmg_train_config;

typedef struct apmg_train_state apmg_train_state;

/* Element offsets of [grids_cl | w1 | w2 | w3 | end] in the flat main-parameter
 * buffer used by the training loop (sections aligned to 64 elements). */
int apmg_main_layout(const apmg_model* m, int64_t offsets[5]);

size_t apmg_train_workspace_bytes(const apmg_model* m, const apmg_train_config* cfg);
/* Extra workspace bytes for the session's private sampler copy of a (w, h, d) volume: add them to
 * apmg_train_workspace_bytes and the copy is carved from the caller's workspace (so the caller's
 * allocator owns and can reuse it); without them the session takes the copy from the library's
 * block cache.  0 when no copy would be made. */
size_t apmg_train_volume_bytes(int32_t w, int32_t h, int32_t d);
/* Parameters are updated in place: grad-free main group `main_params` laid out
 * [grids_cl | w1 | w2 | w3] and `transforms` [M][4][4] (both dtype, device).
 * bias_table: HOST f64 [iterations][2] = (1-0.9^t, 1-0.99^t) for t = 1..iterations
 * computed in Python so Adam's bias corrections match the reference bit for bit.
 * The state samples targets from a private copy of `volume` (corner-replicated cells, or 8^3
 * bricks; see apmg_train_volume_bytes) taken from the tail of `workspace` when it is large enough,
 * else from the library's block cache (returned at apmg_train_destroy). */
int apmg_train_create(apmg_train_state** out, const apmg_model* shape, void* main_params, void* transforms,
                      const float* volume, int32_t w, int32_t h, int32_t d, const apmg_train_config* cfg,
                      const double* bias_table, void* workspace, size_t workspace_bytes, void* stream);
/* enqueue up to n iterations (asynchronous; iterations after a plateau stop are no-ops) */
int apmg_train_run(apmg_train_state* s, int64_t n, void* stream);
/* synchronising: iterations_run and whether the loop has ended */
int apmg_train_status(apmg_train_state* s, int64_t* iterations_run, int32_t* finished, void* stream);
/* synchronising: copy the log (HOST buffers of length >= iterations; triggers >= plateau_max_triggers) */
int apmg_train_log(apmg_train_state* s, double* l_rec, double* l_density, double* lr, int64_t* stop_iteration,
                   int64_t* triggers, int64_t* n_triggers, void* stream);
int apmg_train_destroy(apmg_train_state* s);
/* Adam moments of the session (replaces reading optim.py:38-44 AdamState.m / .v after
 * trainer.py:190-204): device copies into main_m / main_v (apmg_main_layout, grids channel-last)
 * and tf_m / tf_v ((grids, 4, 4)); null destinations are skipped.  Stream-ordered. */
int apmg_train_moments(apmg_train_state* s, void* main_m, void* main_v, void* tf_m, void* tf_v, void* stream);

/* clock64 stamps [16 tiles][8 phases] of CTA 0 of the last tensor-core lattice sweep run with
 * APMG_INFER_STAMPS=1 (profiling aid, tools/infer_phases.py) */
int apmg_debug_infer_phases(long long* out);
/* same for the bf16x3 recon kernel: [16 tiles][12 phases] (APMG_TC_STAMPS=1, tools/tc16_phases.py) */
int apmg_debug_tc16_phases(long long* out);
/* per warp of CTA 0: [16 tiles][16 warps][16 points] (APMG_TC_STAMPS=1, tools/tc16_warps.py) */
int apmg_debug_tc16_warp_phases(long long* out);

/* ---- host-side restatement hooks (unit tests of the scheduler on CPU) -------- */
/* plateau_step (trainer.py:118-138) on the same code the device controller runs.
 * history: HOST ring of capacity window+1 (in/out), count in/out; returns 0 none,
 * 1 reduce_lr, 2 stop. */
int apmg_host_plateau_step(double* history, int64_t* count, int64_t* triggers, int64_t window,
                           double threshold, int64_t max_triggers, double current_ma);
/* transform_stop_check (trainer.py:141-157) */
int apmg_host_transform_stop(const double* history, int64_t count, int64_t window, double threshold,
                             int64_t hard_stop_iteration, int64_t iteration);
/* numpy's pairwise float64 summation (used for every moving average above) */
double apmg_host_pairwise_sum(const double* x, int64_t n);

#ifdef __cplusplus
}
#endif
#endif /* APMG_CUDA_H */
