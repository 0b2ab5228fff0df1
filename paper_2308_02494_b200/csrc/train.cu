// Device-resident training loop: train_single (trainer.py:160-223) with the
// whole control flow -- delayed start, transform stop rule, plateau scheduler,
// masked Adam on both parameter groups -- executed on the GPU so iterations
// are enqueued back to back with no host synchronisation.
//
// Per iteration (all kernels read TrainCtl.skip; density kernels also read
// TrainCtl.density_on):
//   ctl_begin   it, Adam scalars, transform stop decision      (trainer.py:194-201)
//   batch       Philox coords -> fp64 targets -> f32 coords     (trainer.py:189-191)
//   recon       fused encode + MLP fwd/bwd + grid scatter       (optim.py:102-155)
//   recon_fin   dW reduction, l_rec                             (optim.py:118)
//   adam_main   masked Adam, clears grads                       (optim.py:47-73)
//   density x6  rho, stats, target, stats, grad, finalize+Adam  (optim.py:158-200)
//   ctl_end     log, density history, plateau rule              (trainer.py:207-220)
#include <math.h>
#include <stdlib.h>

#include <vector>

#include <chrono>
#include <mutex>

#include "kernels.cuh"
#include "sched.cuh"

namespace apmg {

template <typename T>
__global__ void k_train_batch(uint64_t k0, uint64_t k1, int64_t batch, const float* __restrict__ vol, int w, int h,
                              int d, T* __restrict__ coords, T* __restrict__ targets, const TrainCtl* ctl);
template <typename T>
__global__ void k_adam_train(T* __restrict__ p, T* __restrict__ g, T* __restrict__ m, T* __restrict__ v, int64_t n,
                             const TrainCtl* ctl, float* __restrict__ gx, int64_t gx_elems, int qw,
                             float* __restrict__ dgx, unsigned long long* __restrict__ gfx, int64_t fx_elems);
constexpr int kBuckets = 32768;
__global__ void k_batch_keys(uint64_t k0, uint64_t k1, int64_t batch, double* __restrict__ c64,
                             uint32_t* __restrict__ key, int32_t* __restrict__ counts, const TrainCtl* ctl);
__global__ void k_bucket_scan(int32_t* __restrict__ counts, const TrainCtl* ctl, int ahead);
__global__ void k_batch_keys_cells(uint64_t k0, uint64_t k1, int64_t batch, const float4* __restrict__ cells, int w,
                                   int h, int d, float4* __restrict__ rec, uint32_t* __restrict__ key,
                                   int32_t* __restrict__ counts, const TrainCtl* ctl, int ahead);
__global__ void k_bucket_scatter_rec(const float4* __restrict__ rec, const uint32_t* __restrict__ key, int64_t n,
                                     int32_t* __restrict__ cursor, float* __restrict__ coords,
                                     float* __restrict__ targets, const TrainCtl* ctl, int ahead,
                                     float2* __restrict__ tA, float2* __restrict__ tB, int32_t* __restrict__ perm);
__global__ void k_bucket_stable_rec(const float2* __restrict__ tA, const float2* __restrict__ tB,
                                    const int32_t* __restrict__ perm, const int32_t* __restrict__ end, int nbuckets,
                                    float* __restrict__ coords, float* __restrict__ targets, const TrainCtl* ctl,
                                    int ahead);
__global__ void k_bucket_scatter(const double* __restrict__ c64, const uint32_t* __restrict__ key, int64_t n,
                                 int32_t* __restrict__ cursor, double* __restrict__ c64_out,
                                 int32_t* __restrict__ perm, const TrainCtl* ctl);
__global__ void k_bucket_stable(const double* __restrict__ c64_in, const int32_t* __restrict__ perm,
                                const int32_t* __restrict__ end, int nbuckets, double* __restrict__ c64_out,
                                const TrainCtl* ctl);
template <typename T>
__global__ void k_sample_sorted(const double* __restrict__ c64, int64_t n, const float* __restrict__ vol, int w,
                                int h, int d, T* __restrict__ coords, T* __restrict__ targets, const TrainCtl* ctl);
__global__ void k_brick_volume(const float* __restrict__ vol, int w, int h, int d, int nbx, int nby,
                               float* __restrict__ out);
template <typename T>
__global__ void k_sample_sorted_bricked(const double* __restrict__ c64, int64_t n, const float* __restrict__ bricks,
                                        int w, int h, int d, int nbx, int nby, T* __restrict__ coords,
                                        T* __restrict__ targets, const TrainCtl* ctl);

__global__ void k_cell_volume(const float* __restrict__ vol, int w, int h, int d, float4* __restrict__ out);
template <typename T>
__global__ void k_sample_sorted_cells(const double* __restrict__ c64, int64_t n, const float4* __restrict__ cells,
                                      int w, int h, int d, T* __restrict__ coords, T* __restrict__ targets,
                                      const TrainCtl* ctl);

static bool sort_enabled() {
  const char* e = getenv("APMG_SORT");
  return !(e && e[0] == '0');
}

struct CtlParams {
  int64_t iterations, delay_start, ma_window, hard_stop, plateau_window, plateau_max;
  double lr_main, lr_tf, improve_thr, plateau_thr, plateau_factor;
  int32_t plateau_enabled;
};

__global__ void k_ctl_begin(TrainCtl* ctl, CtlParams P, const double* __restrict__ dens_hist,
                            const double* __restrict__ bias) {
  if (threadIdx.x != 0) return;
  if (ctl->finished) {
    ctl->skip = 1;
    ctl->gen_skip = 1;
    return;
  }
  ctl->skip = 0;
  const int64_t it = ctl->it;
  ctl->gen_it = it + 1;
  ctl->gen_skip = it + 1 >= P.iterations ? 1 : 0;
  const int64_t tm = ++ctl->t_main;
  ctl->lr_main_t = P.lr_main * ctl->lr_scale;
  ctl->bc1_main = bias[2 * (tm - 1)];
  ctl->bc2_main = bias[2 * (tm - 1) + 1];
  ctl->density_on = 0;
  if (ctl->transforms_active && it >= P.delay_start) {
    if (transform_stop_rule(dens_hist, ctl->dens_count, P.ma_window, P.improve_thr, P.hard_stop, it)) {
      ctl->transforms_active = 0;
      ctl->stop_iteration = it;
    } else {
      ctl->density_on = 1;
      const int64_t tt = ++ctl->t_tf;
      ctl->lr_tf_t = P.lr_tf * ctl->lr_scale;
      ctl->bc1_tf = bias[2 * (tt - 1)];
      ctl->bc2_tf = bias[2 * (tt - 1) + 1];
    }
  }
}

__global__ void k_ctl_end(TrainCtl* ctl, CtlParams P, const double* __restrict__ l_rec_log, double* l_dens_log,
                          double* lr_log, double* dens_hist, double* plat_ring, int64_t* trig_log) {
  if (threadIdx.x != 0 || ctl->skip) return;
  const int64_t it = ctl->it;
  if (ctl->density_on) {
    l_dens_log[it] = ctl->l_dens;
    dens_hist[ctl->dens_count++] = ctl->l_dens;
  } else {
    l_dens_log[it] = __longlong_as_double(0x7ff8000000000000ll);  // None
  }
  lr_log[it] = P.lr_main * ctl->lr_scale;
  ctl->iterations_run = it + 1;
  if (P.plateau_enabled && it + 1 >= P.plateau_window) {
    const double ma = ring_pairwise_sum(l_rec_log, P.iterations, it + 1 - P.plateau_window, P.plateau_window) /
                      double(P.plateau_window);
    const int64_t before = ctl->n_triggers;
    const int act = plateau_step_rule(plat_ring, &ctl->plat_count, &ctl->n_triggers, P.plateau_window,
                                      P.plateau_thr, P.plateau_max, ma);
    if (act) {
      trig_log[before] = it;
      ctl->lr_scale /= P.plateau_factor;
      if (act == 2) ctl->finished = 1;
    }
  }
  ctl->it = it + 1;
  if (it + 1 >= P.iterations) ctl->finished = 1;
}

}  // namespace apmg

using namespace apmg;

struct apmg_train_state {
  apmg_model shape;
  apmg_train_config cfg;
  CtlParams P;
  void* main_params;
  void* transforms;
  const float* volume;
  int w, h, d;
  int64_t off[5];
  TrainCtl* ctl;
  double *l_rec, *l_dens, *lr, *dens_hist, *plat_ring, *bias;
  int64_t* trig;
  void *grad, *am, *av, *tm, *tv, *coords, *targets, *sq;
  double *c64_raw, *c64_sorted;  // sorted path: f64 batch coordinates before / after bucketing
  uint32_t* key;
  int32_t* counts;
  bool sort;
  void* recon_ws;
  size_t recon_wsb;
  void* dens_ws;
  size_t dens_wsb;
  // CUDA graph of kGraphIters iterations, captured on first use and replayed (the
  // iteration sequence is identical every time: all state lives in TrainCtl)
  cudaGraphExec_t graph = nullptr;
  uint64_t graph_launches = 0;
  // 8x8x8-bricked copy of the volume for the sorted sampler (owned; APMG_BRICKED=0 disables)
  float4* gridx = nullptr;  // x-pair grid copy (ModelDev::gridx), or null
  unsigned long long* gfx = nullptr;  // deterministic mode: fixed-point grid gradient [grid elements]
  int32_t* perm = nullptr;            // deterministic mode: batch index of each bucketed point
  int64_t fx_elems = 0;
  float4* gradx = nullptr;  // x-pair grid gradient (ModelDev::grad_pairs), or null
  int64_t gx_cells = 0;
  int gq_w = 0;  // > 0: gridx holds the xy-quad copy (ModelDev::gridq; 2 float4 per cell), row width W
  float* vol_bricked = nullptr;
  size_t vol_bricked_bytes = 0;
  bool vol_owned = false;  // from the block cache (returned at destroy), else part of the workspace
  bool vol_cells = false;  // vol_bricked holds the corner-replicated cell copy (k_cell_volume)
  int nbx = 0, nby = 0;
  // fused batch path (float session, corner-replicated volume, float REDs): the next iteration's
  // batch is generated on a side stream while this iteration's Adam and density steps run, into
  // the other of two (coords, targets) buffers (the second carved from c64_sorted, unused there)
  bool fused = false, pipe = false;
  bool adam_side = false;  // masked Adam of the main group on the side stream (pipe only)
  void* coords_b[2] = {nullptr, nullptr};
  void* targets_b[2] = {nullptr, nullptr};
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  bool batch_ready = false;  // the batch of the next iteration to run is in coords_b[host_it & 1]
  int64_t host_it = 0;       // run_one calls so far (buffer parity)
  int64_t graph_parity = 0;  // host_it & 1 when the graph was captured
};

constexpr int64_t kGraphIters = 8;

// The sorted sampler's private copy of the volume: corner-replicated cells (APMG_CELLVOL=0: off;
// 8x the volume, used while that stays within 16 GiB and a quarter of the device memory that is
// free or cached by the block pool) or else 8^3 bricks (APMG_BRICKED=0: off, 1x the volume).
struct SamplerCopy {
  size_t bytes = 0;
  bool cells = false;
};
static SamplerCopy sampler_copy_plan(int32_t w, int32_t h, int32_t d, bool sort) {
  SamplerCopy c;
  if (!sort) return c;
  const char* ec = getenv("APMG_CELLVOL");
  const size_t cell_bytes = size_t(32) * size_t(w > 1 ? w - 1 : 1) * size_t(h > 1 ? h - 1 : 1) *
                            size_t(d > 1 ? d - 1 : 1);
  // free device memory, re-queried at most every 5 s: cudaMemGetInfo took 0.3-70 ms (erratic)
  // when it ran with the session's volume DMA in flight, and this plan is made on every session
  // setup (twice); a quarter of free memory is a coarse budget that a few-seconds-old value serves
  static std::mutex mu;
  static size_t free_cached = 0;
  static std::chrono::steady_clock::time_point t_cached;
  static bool have = false;
  size_t free_b = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    const auto now = std::chrono::steady_clock::now();
    if (!have || now - t_cached > std::chrono::seconds(5)) {
      size_t total_b = 0;
      if (cudaMemGetInfo(&free_cached, &total_b) != cudaSuccess) {
        cudaGetLastError();
        free_cached = 0;
      }
      t_cached = now;
      have = true;
    }
    free_b = free_cached;
  }
  const size_t budget = std::min(size_t(16) << 30, (free_b + pool_cached_bytes()) / 4);
  if (!(ec && ec[0] == '0') && cell_bytes <= budget) {
    c.bytes = cell_bytes;
    c.cells = true;
    return c;
  }
  const char* eb = getenv("APMG_BRICKED");
  if (eb && eb[0] == '0') return c;
  c.bytes = sizeof(float) * 512 * size_t((w + 7) / 8) * size_t((h + 7) / 8) * size_t((d + 7) / 8);
  return c;
}

extern "C" size_t apmg_train_volume_bytes(int32_t w, int32_t h, int32_t d) {
  if (w < 1 || h < 1 || d < 1) return 0;
  return sampler_copy_plan(w, h, d, sort_enabled()).bytes;
}

extern "C" int apmg_main_layout(const apmg_model* m, int64_t offsets[5]) {
  APMG_ARG_CHECK(m != nullptr, "null model");
  const int64_t F = int64_t(m->grids) * m->channels;
  const int64_t G = F * m->depth * m->height * m->width;
  auto al = [](int64_t v) { return (v + 63) / 64 * 64; };
  offsets[0] = 0;
  offsets[1] = al(G);
  offsets[2] = offsets[1] + al(64 * F);
  offsets[3] = offsets[2] + al(64 * 64);
  offsets[4] = offsets[3] + al(64);
  return APMG_OK;
}

static size_t carve_train(apmg_train_state* s, const apmg_model* m, const apmg_train_config* c, void* ws,
                          size_t wsb) {
  const size_t es = m->dtype == APMG_F32 ? 4 : 8;
  int64_t off[5];
  apmg_main_layout(m, off);
  const int64_t iters = std::max<int64_t>(c->iterations, 1), B = c->batch_size;
  const int F = m->grids * m->channels;
  Carver cv(ws, wsb);
  TrainCtl* ctl = cv.take<TrainCtl>(1);
  double* l_rec = cv.take<double>(iters);
  double* l_dens = cv.take<double>(iters);
  double* lr = cv.take<double>(iters);
  double* dens_hist = cv.take<double>(iters);
  double* plat_ring = cv.take<double>(std::max<int64_t>(c->plateau_window + 1, 1));
  double* bias = cv.take<double>(2 * iters);
  int64_t* trig = cv.take<int64_t>(std::max<int64_t>(c->plateau_max_triggers, 1));
  char* grad = cv.take<char>(es * off[4]);
  char* am = cv.take<char>(es * off[4]);
  char* av = cv.take<char>(es * off[4]);
  char* tm = cv.take<char>(es * 16 * m->grids);
  char* tv = cv.take<char>(es * 16 * m->grids);
  char* coords = cv.take<char>(es * 3 * B);
  char* targets = cv.take<char>(es * B);
  char* sq = cv.take<char>(es * B);
  double* c64_raw = cv.take<double>(3 * B);
  double* c64_sorted = cv.take<double>(3 * B);
  uint32_t* key = cv.take<uint32_t>(B);
  int32_t* counts = cv.take<int32_t>(kBuckets);
  const size_t rws = m->dtype == APMG_F32 ? recon_ws_bytes<float>(F, B) : recon_ws_bytes<double>(F, B);
  char* recon_ws = cv.take<char>(rws);
  const size_t dws = density_ws_bytes(m->grids, B);
  char* dens_ws = cv.take<char>(dws);
  // x-pair grid copy for the tensor-core encoder (two-channel f32 models; APMG_GRIDX=0 off)
  const char* eg = getenv("APMG_GRIDX");
  const bool use_gx = m->dtype == APMG_F32 && m->channels == 2 && !(eg && eg[0] == '0');
  const int64_t cells = int64_t(m->grids) * m->depth * m->height * m->width;
  // ... as the xy-quad copy where the tensor-core recon kernel reads it (two 256-bit gathers per
  // (point, grid) instead of four 128-bit ones, a group's 8 in flight: 1.413 -> 1.369 ms per
  // launch; masked Adam's four copy writes per cell run on the side stream, hidden behind the
  // density step). APMG_GRIDQ=0: the x-pair copy
  const char* eq = getenv("APMG_GRIDQ");
  const bool use_gq = use_gx && recon_uses_tc16(*m) && !(eq && eq[0] == '0');
  float4* gridx = use_gx ? cv.take<float4>(use_gq ? 2 * cells : cells) : nullptr;
  // ... and the x-pair grid gradient when the bf16x3 recon kernel runs (APMG_GRADX=0 off)
  const char* ed = getenv("APMG_GRADX");
  const bool det = c->deterministic != 0;
  const bool use_dgx = use_gx && recon_uses_tc16(*m) && !(ed && ed[0] == '0') && !det;
  float4* gradx = use_dgx ? cv.take<float4>(cells) : nullptr;
  const int64_t gel = cells * m->channels;
  unsigned long long* gfx = det ? cv.take<unsigned long long>(gel) : nullptr;
  int32_t* perm = det ? cv.take<int32_t>(B) : nullptr;
  if (s) {
    s->gfx = gfx;
    s->perm = perm;
    s->fx_elems = det ? gel : 0;
    s->gridx = gridx;
    s->gradx = gradx;
    s->gx_cells = use_gx ? cells : 0;
    s->gq_w = use_gq ? m->width : 0;
    s->ctl = ctl;
    s->l_rec = l_rec;
    s->l_dens = l_dens;
    s->lr = lr;
    s->dens_hist = dens_hist;
    s->plat_ring = plat_ring;
    s->bias = bias;
    s->trig = trig;
    s->grad = grad;
    s->am = am;
    s->av = av;
    s->tm = tm;
    s->tv = tv;
    s->coords = coords;
    s->targets = targets;
    s->sq = sq;
    s->c64_raw = c64_raw;
    s->c64_sorted = c64_sorted;
    s->key = key;
    s->counts = counts;
    s->recon_ws = recon_ws;
    s->recon_wsb = rws;
    s->dens_ws = dens_ws;
    s->dens_wsb = dws;
    for (int i = 0; i < 5; ++i) s->off[i] = off[i];
  }
  return cv.used + 256;
}

extern "C" size_t apmg_train_workspace_bytes(const apmg_model* m, const apmg_train_config* cfg) {
  if (!m || !cfg) return 0;
  return carve_train(nullptr, m, cfg, nullptr, 0);
}

extern "C" int apmg_train_create(apmg_train_state** out, const apmg_model* shape, void* main_params, void* transforms,
                                 const float* volume, int32_t w, int32_t h, int32_t d, const apmg_train_config* cfg,
                                 const double* bias_table, void* workspace, size_t workspace_bytes, void* stream) {
  APMG_ARG_CHECK(out && shape && cfg && main_params && transforms && volume, "null argument");
  APMG_ARG_CHECK(shape->dtype == APMG_F32 || shape->dtype == APMG_F64, "bad dtype");
  APMG_ARG_CHECK(shape->hidden == 64, "hidden width must be 64");
  APMG_ARG_CHECK(cfg->iterations >= 1 && cfg->batch_size >= 1, "iterations and batch_size must be >= 1");
  APMG_ARG_CHECK(cfg->plateau_window >= 1 && cfg->transform_ma_window >= 1, "windows must be positive");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  apmg_train_state* s = new apmg_train_state();
  s->shape = *shape;
  s->cfg = *cfg;
  s->main_params = main_params;
  s->transforms = transforms;
  s->volume = volume;
  s->w = w;
  s->h = h;
  s->d = d;
  s->sort = sort_enabled();
  const size_t need = carve_train(s, shape, cfg, workspace, workspace_bytes);
  if (need > workspace_bytes) {
    delete s;
    set_error("train workspace too small: need %zu have %zu", need, workspace_bytes);
    return APMG_E_WORKSPACE;
  }
  {
    // sampler copy of the volume: carved from the caller's workspace when it was sized with
    // apmg_train_volume_bytes (torch's caching allocator then owns the block), else from the
    // library's block cache
    const SamplerCopy sc = sampler_copy_plan(w, h, d, s->sort);
    const size_t tail = (need + 255) / 256 * 256;
    if (sc.bytes && workspace_bytes >= tail + sc.bytes) {
      s->vol_bricked = reinterpret_cast<float*>(static_cast<char*>(workspace) + tail);
      s->vol_owned = false;
    } else if (sc.bytes) {
      s->vol_bricked = static_cast<float*>(pool_alloc(sc.bytes));
      s->vol_owned = true;
    }
    if (s->vol_bricked) {
      s->vol_bricked_bytes = sc.bytes;
      if (sc.cells) {
        s->vol_cells = true;
        const int64_t nc = int64_t(sc.bytes / 32);
        const int g = int(std::min<int64_t>(ceil_div(nc, 256), int64_t(num_sms()) * 32));
        APMG_LAUNCH("cell_volume", k_cell_volume, g, 256, 0, st, volume, w, h, d,
                    reinterpret_cast<float4*>(s->vol_bricked));
      } else {
        s->nbx = (w + 7) / 8;
        s->nby = (h + 7) / 8;
        const int64_t nv = int64_t(w) * h * d;
        const int g = int(std::min<int64_t>(ceil_div(nv, 256), int64_t(num_sms()) * 32));
        APMG_LAUNCH("brick_volume", k_brick_volume, g, 256, 0, st, volume, w, h, d, s->nbx, s->nby, s->vol_bricked);
      }
    }  // else no copy (sorting off, APMG_BRICKED=0, or no room): sample the row-major volume
  }
  {
    const char* efb = getenv("APMG_FUSED_BATCH");
    const char* ep = getenv("APMG_BATCH_AHEAD");
    // (deterministic sessions too: their batch is put back in batch order inside each bucket)
    s->fused = s->sort && shape->dtype == APMG_F32 && s->vol_cells && !(efb && efb[0] == '0');
    s->pipe = s->fused && !(ep && ep[0] == '0');
    const char* ea = getenv("APMG_ADAM_SIDE");
    s->adam_side = s->pipe && !(ea && ea[0] == '0');
    s->coords_b[0] = s->coords;
    s->targets_b[0] = s->targets;
    if (s->pipe) {
      const int64_t B = cfg->batch_size;
      s->coords_b[1] = s->c64_sorted;                                   // 12 B of its 24 B per point
      s->targets_b[1] = reinterpret_cast<float*>(s->c64_sorted) + 3 * B;  // + 4 B
      APMG_CUDA_TRY(cudaStreamCreateWithFlags(&s->side, cudaStreamNonBlocking));
      APMG_CUDA_TRY(cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming));
      APMG_CUDA_TRY(cudaEventCreateWithFlags(&s->ev_join, cudaEventDisableTiming));
    }
  }
  CtlParams& P = s->P;
  P.iterations = cfg->iterations;
  P.delay_start = cfg->delay_start;
  P.ma_window = cfg->transform_ma_window;
  P.hard_stop = cfg->hard_stop_iteration;
  P.plateau_window = cfg->plateau_window;
  P.plateau_max = cfg->plateau_max_triggers;
  P.lr_main = cfg->lr_main;
  P.lr_tf = cfg->lr_transform;
  P.improve_thr = cfg->transform_improve_threshold;
  P.plateau_thr = cfg->plateau_threshold;
  P.plateau_factor = cfg->plateau_factor;
  P.plateau_enabled = cfg->plateau_enabled;
  TrainCtl c{};
  c.transforms_active = cfg->train_transforms ? 1 : 0;
  c.stop_iteration = -1;
  c.lr_scale = 1.0;
  const size_t es = shape->dtype == APMG_F32 ? 4 : 8;
  APMG_CUDA_TRY(cudaMemcpyAsync(s->ctl, &c, sizeof(c), cudaMemcpyHostToDevice, st));
  APMG_CUDA_TRY(cudaMemcpyAsync(s->bias, bias_table, sizeof(double) * 2 * cfg->iterations, cudaMemcpyHostToDevice, st));
  APMG_CUDA_TRY(cudaMemsetAsync(s->grad, 0, es * s->off[4], st));
  if (s->gradx) APMG_CUDA_TRY(cudaMemsetAsync(s->gradx, 0, sizeof(float4) * s->gx_cells, st));
  if (s->gfx) APMG_CUDA_TRY(cudaMemsetAsync(s->gfx, 0, sizeof(unsigned long long) * s->fx_elems, st));
  APMG_CUDA_TRY(cudaMemsetAsync(s->am, 0, es * s->off[4], st));
  APMG_CUDA_TRY(cudaMemsetAsync(s->av, 0, es * s->off[4], st));
  APMG_CUDA_TRY(cudaMemsetAsync(s->tm, 0, es * 16 * shape->grids, st));
  APMG_CUDA_TRY(cudaMemsetAsync(s->tv, 0, es * 16 * shape->grids, st));
  APMG_CUDA_TRY(cudaMemsetAsync(s->l_rec, 0, sizeof(double) * cfg->iterations, st));
  APMG_CUDA_TRY(cudaStreamSynchronize(st));  // bias_table / ctl host staging
  *out = s;
  return APMG_OK;
}

template <typename T>
static int run_one(apmg_train_state* s, cudaStream_t st) {
  const apmg_model& m = s->shape;
  const apmg_train_config& c = s->cfg;
  const int64_t B = c.batch_size;
  T* params = static_cast<T*>(s->main_params);
  T* grad = static_cast<T*>(s->grad);
  apmg_model live = m;
  live.grids_cl = params + s->off[0];
  live.w1 = params + s->off[1];
  live.w2 = params + s->off[2];
  live.w3 = params + s->off[3];
  live.transforms = s->transforms;
  ModelDev<T> md = make_model_dev<T>(live);
  md.gridx = s->gq_w ? nullptr : s->gridx;
  md.gridq = s->gq_w ? reinterpret_cast<const float*>(s->gridx) : nullptr;
  md.grad_pairs = s->gradx != nullptr;
  md.dgrid_fx = s->gfx;
  // density pass fused into the recon kernel (APMG_FUSED_RHO=0: separate rho kernel, A/B)
  int pre_nb = 0;
  if constexpr (sizeof(T) == 4) {
    const char* ef = getenv("APMG_FUSED_RHO");
    const char* e64 = getenv("APMG_DENSITY64");
    const char* ex2 = getenv("APMG_DENSITY_X2");
    if (c.train_transforms && m.flat_top_p == 10 && recon_uses_tc16(live) && !(ef && ef[0] == '0') &&
        !(e64 && e64[0] == '1') && !(ex2 && ex2[0] == '0')) {
      if (int rc = density_rho_slots(m.grids, B, s->dens_ws, s->dens_wsb, &md.rho_out, &md.rho_part)) return rc;
      pre_nb = recon_tc16_grid(B);
    }
  }
  APMG_LAUNCH("ctl_begin", k_ctl_begin, 1, 32, 0, st, s->ctl, s->P, s->dens_hist, s->bias);
  // this iteration's batch buffers (two alternate when the next batch is generated ahead)
  const int cur = s->pipe ? int(s->host_it & 1) : 0;
  T* coords = static_cast<T*>(s->coords_b[cur]);
  T* targets = static_cast<T*>(s->targets_b[cur]);
  // float session, corner-replicated volume, default (float-RED) mode: targets sampled with the
  // batch, (x, y, z, target) records bucketed straight into the recon inputs; ahead = 1 generates
  // the batch of iteration it + 1 (TrainCtl::gen_it)
  auto fused_batch = [&](cudaStream_t bs, int ahead, void* cx, void* tx) -> int {
    APMG_CUDA_TRY(cudaMemsetAsync(s->counts, 0, sizeof(int32_t) * kBuckets, bs));
    float4* rec = reinterpret_cast<float4*>(s->c64_raw);  // 16 of its 24 bytes per point
    APMG_LAUNCH("batch_keys", k_batch_keys_cells, elementwise_grid(B, 8), 256, 0, bs, c.key0, c.key1, B,
                reinterpret_cast<const float4*>(s->vol_bricked), s->w, s->h, s->d, rec, s->key, s->counts, s->ctl,
                ahead);
    APMG_LAUNCH("bucket_scan", k_bucket_scan, 1, 1024, 0, bs, s->counts, s->ctl, ahead);
    if (s->perm) {
      // deterministic mode: records and batch indices into the unused tails of the two c64 buffers
      // (floats [4B, 6B) of each; the records use [0, 4B) of c64_raw, the ahead batch [0, 4B) of
      // c64_sorted), then each bucket back in batch order into the recon inputs
      float2* tA = reinterpret_cast<float2*>(reinterpret_cast<float*>(s->c64_raw) + 4 * B);
      float2* tB = reinterpret_cast<float2*>(reinterpret_cast<float*>(s->c64_sorted) + 4 * B);
      APMG_LAUNCH("bucket_scatter", k_bucket_scatter_rec, elementwise_grid(B, 8), 256, 0, bs, rec, s->key, B,
                  s->counts, nullptr, nullptr, s->ctl, ahead, tA, tB, s->perm);
      APMG_LAUNCH("bucket_stable", k_bucket_stable_rec, int(ceil_div(int64_t(kBuckets) * 32, 256)), 256, 0, bs, tA,
                  tB, s->perm, s->counts, kBuckets, static_cast<float*>(cx), static_cast<float*>(tx), s->ctl, ahead);
      return APMG_OK;
    }
    APMG_LAUNCH("bucket_scatter", k_bucket_scatter_rec, elementwise_grid(B, 8), 256, 0, bs, rec, s->key, B,
                s->counts, static_cast<float*>(cx), static_cast<float*>(tx), s->ctl, ahead, nullptr, nullptr, nullptr);
    return APMG_OK;
  };
  if (s->fused && sizeof(T) == 4) {
    if (!(s->pipe && s->batch_ready))
      if (int rc = fused_batch(st, 0, coords, targets)) return rc;
  } else if (s->sort) {
    // batch -> spatial buckets (Morton order) -> permuted batch consumed by recon and density
    APMG_CUDA_TRY(cudaMemsetAsync(s->counts, 0, sizeof(int32_t) * kBuckets, st));
    APMG_LAUNCH("batch_keys", k_batch_keys, elementwise_grid(B, 8), 256, 0, st, c.key0, c.key1, B, s->c64_raw, s->key,
                s->counts, s->ctl);
    APMG_LAUNCH("bucket_scan", k_bucket_scan, 1, 1024, 0, st, s->counts, s->ctl, 0);
    APMG_LAUNCH("bucket_scatter", k_bucket_scatter, elementwise_grid(B, 8), 256, 0, st, s->c64_raw, s->key, B,
                s->counts, s->c64_sorted, s->perm, s->ctl);
    const double* sorted = s->c64_sorted;
    if (s->perm) {  // deterministic mode: batch order within each bucket (c64_raw is free by now)
      APMG_LAUNCH("bucket_stable", k_bucket_stable, int(ceil_div(int64_t(kBuckets) * 32, 256)), 256, 0, st,
                  s->c64_sorted, s->perm, s->counts, kBuckets, s->c64_raw, s->ctl);
      sorted = s->c64_raw;
    }
    if (s->vol_cells)
      APMG_LAUNCH("train_batch", k_sample_sorted_cells<T>, elementwise_grid(B, 8), 256, 0, st, sorted, B,
                  reinterpret_cast<const float4*>(s->vol_bricked), s->w, s->h, s->d, coords,
                  targets, s->ctl);
    else if (s->vol_bricked)
      APMG_LAUNCH("train_batch", k_sample_sorted_bricked<T>, elementwise_grid(B, 8), 256, 0, st, sorted, B,
                  s->vol_bricked, s->w, s->h, s->d, s->nbx, s->nby, coords,
                  targets, s->ctl);
    else
      APMG_LAUNCH("train_batch", k_sample_sorted<T>, elementwise_grid(B, 8), 256, 0, st, sorted, B,
                  s->volume, s->w, s->h, s->d, coords, targets, s->ctl);
  } else {
    APMG_LAUNCH("train_batch", k_train_batch<T>, elementwise_grid(B, 8), 256, 0, st, c.key0, c.key1, B, s->volume,
                s->w, s->h, s->d, coords, targets, s->ctl);
  }
  int rc = launch_recon<T>(md, B, coords, targets,
                           static_cast<T*>(s->sq), nullptr,
                           s->gradx ? reinterpret_cast<T*>(s->gradx) : grad + s->off[0], grad + s->off[1],
                           grad + s->off[2],
                           grad + s->off[3], s->recon_ws, s->recon_wsb, s->ctl, s->l_rec, st);
  if (rc) return rc;
  auto adam_main = [&](cudaStream_t as) -> int {
    APMG_LAUNCH("adam_main", k_adam_train<T>, elementwise_grid(s->off[4], 8), 256, 0, as, params, grad,
                static_cast<T*>(s->am), static_cast<T*>(s->av), s->off[4], s->ctl,
                reinterpret_cast<float*>(s->gridx), 2 * s->gx_cells, s->gq_w, reinterpret_cast<float*>(s->gradx),
                s->gfx, s->fx_elems);
    return APMG_OK;
  };
  bool adam_done = false;
#ifdef APMG_ABL_FREEZE  // timing builds only: parameters frozen (no Adam, no density step), so
  // ablated kernels computing wrong values cannot change later iterations' inputs
  adam_done = m.grids > 0;
#endif
  if (s->pipe && sizeof(T) == 4) {
    // side stream, after the recon (and its finalize: the gradients): the next iteration's batch,
    // then masked Adam on the main group -- both concurrent with the density step on this stream
    // (Adam reads nothing the density step writes; it is memory-bound, the density gradient FP32)
    APMG_CUDA_TRY(cudaEventRecord(s->ev_fork, st));
    APMG_CUDA_TRY(cudaStreamWaitEvent(s->side, s->ev_fork, 0));
    if (int rc2 = fused_batch(s->side, 1, s->coords_b[cur ^ 1], s->targets_b[cur ^ 1])) return rc2;
    if (!adam_done && s->adam_side && !kernel_timing_on()) {  // per-kernel timing: inline (its own time)
      if (int rc2 = adam_main(s->side)) return rc2;
      adam_done = true;
    }
    APMG_CUDA_TRY(cudaEventRecord(s->ev_join, s->side));
  }
  // end of the iteration: join the side stream (the next iteration's recon reads the batch and
  // the parameters it wrote; the controller may change the learning rate Adam read), controller
  auto finish = [&]() -> int {
    if (s->pipe && sizeof(T) == 4) {
      APMG_CUDA_TRY(cudaStreamWaitEvent(st, s->ev_join, 0));
      s->batch_ready = true;
    }
    APMG_LAUNCH("ctl_end", k_ctl_end, 1, 32, 0, st, s->ctl, s->P, s->l_rec, s->l_dens, s->lr, s->dens_hist,
                s->plat_ring, s->trig);
    ++s->host_it;
    return APMG_OK;
  };
#ifdef APMG_ABL_FREEZE
  if (m.grids > 0) return finish();
#endif
  if (!adam_done)
    if (int rc2 = adam_main(st)) return rc2;
  if (c.train_transforms) {
    rc = launch_density<T, T>(static_cast<T*>(s->transforms), m.grids, m.flat_top_p, coords,
                              static_cast<const T*>(s->sq), B, nullptr, nullptr, nullptr, static_cast<T*>(s->tm),
                              static_cast<T*>(s->tv), s->dens_ws, s->dens_wsb, s->ctl, st, pre_nb);
    if (rc) return rc;
  }
  return finish();
}

static int run_direct(apmg_train_state* s, cudaStream_t st) {
  return s->shape.dtype == APMG_F32 ? run_one<float>(s, st) : run_one<double>(s, st);
}

static bool graphs_enabled() {
  const char* e = getenv("APMG_GRAPH");  // APMG_GRAPH=0: plain launches (A/B, debugging)
  return !(e && e[0] == '0') && !kernel_timing_on();
}

extern "C" int apmg_train_run(apmg_train_state* s, int64_t n, void* stream) {
  APMG_ARG_CHECK(s != nullptr, "null state");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int64_t done = 0;
  if (s->gridx && n > 0) {  // (re)build the grid copy: the caller may have rewritten the parameters
    const float2* g2 = reinterpret_cast<const float2*>(static_cast<float*>(s->main_params) + s->off[0]);
    if (s->gq_w)
      APMG_LAUNCH("pack_gridq", k_pack_gridq, elementwise_grid(s->gx_cells, 8), 256, 0, st, g2, s->gridx, s->gx_cells,
                  s->gq_w);
    else
      APMG_LAUNCH("pack_gridx", k_pack_gridx, elementwise_grid(s->gx_cells, 8), 256, 0, st, g2, s->gridx,
                  s->gx_cells);
  }
  // the graph is captured as soon as the session will replay it (a short first call -- a warm-up --
  // captures it too, so a later timed call does not pay the capture); capturing runs nothing
  const bool will_replay = n >= kGraphIters || s->cfg.iterations >= 2 * kGraphIters;
  if (graphs_enabled() && !(s->cfg.reserved & 1) && will_replay && n >= 1) {
    if (!s->graph) {
      int rc = run_direct(s, st);  // first iteration direct: one-time launch attributes set outside capture
      if (rc) return rc;
      ++done;
      // capture on a private stream (the caller's may be the legacy default stream, which
      // cannot capture); the graph is replayed on the caller's stream
      cudaStream_t cs = nullptr;
      APMG_CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
      APMG_CUDA_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed));
      const uint64_t c0 = launch_counter().load();
      s->graph_parity = s->host_it & 1;
      for (int64_t i = 0; i < kGraphIters && rc == 0; ++i) rc = run_direct(s, cs);
      cudaGraph_t g = nullptr;
      const cudaError_t ec = cudaStreamEndCapture(cs, &g);
      cudaStreamDestroy(cs);
      s->graph_launches = launch_counter().load() - c0;
      launch_counter().fetch_sub(s->graph_launches);  // counted when replayed
      if (rc) {
        if (g) cudaGraphDestroy(g);
        return rc;
      }
      if (ec != cudaSuccess) {
        set_error("train graph capture: %s", cudaGetErrorString(ec));
        return APMG_E_CUDA;
      }
      const cudaError_t ei = cudaGraphInstantiate(&s->graph, g, 0);
      cudaGraphDestroy(g);
      if (ei != cudaSuccess) {
        s->graph = nullptr;
        set_error("train graph instantiate: %s", cudaGetErrorString(ei));
        return APMG_E_CUDA;
      }
    }
    // the graph's buffer parity is fixed at capture (kGraphIters is even): one direct iteration
    // realigns after an odd number of direct ones
    if (s->pipe && (s->host_it & 1) != s->graph_parity && n - done > kGraphIters) {
      if (int rc = run_direct(s, st)) return rc;
      ++done;
    }
    for (; n - done >= kGraphIters && (!s->pipe || (s->host_it & 1) == s->graph_parity); done += kGraphIters) {
      APMG_CUDA_TRY(cudaGraphLaunch(s->graph, st));
      launch_counter().fetch_add(s->graph_launches);
      s->host_it += kGraphIters;
    }
  }
  for (; done < n; ++done) {
    const int rc = run_direct(s, st);
    if (rc) return rc;
  }
  return APMG_OK;
}

extern "C" int apmg_train_status(apmg_train_state* s, int64_t* iterations_run, int32_t* finished, void* stream) {
  APMG_ARG_CHECK(s != nullptr, "null state");
  TrainCtl c;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  APMG_CUDA_TRY(cudaMemcpyAsync(&c, s->ctl, sizeof(c), cudaMemcpyDeviceToHost, st));
  APMG_CUDA_TRY(cudaStreamSynchronize(st));
  if (iterations_run) *iterations_run = c.iterations_run;
  if (finished) *finished = c.finished;
  return APMG_OK;
}

// Adam state of the session (optim.py:38-44 AdamState: the m / v moments) -- checkpointing and
// parity inspection.  Device-to-device copies on `stream`; main_m / main_v take the main group's
// flat layout (apmg_main_layout, grids channel-last), tf_m / tf_v the (grids, 4, 4) transforms.
// Any destination may be null.
extern "C" int apmg_train_moments(apmg_train_state* s, void* main_m, void* main_v, void* tf_m, void* tf_v,
                                  void* stream) {
  APMG_ARG_CHECK(s != nullptr, "null state");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t es = s->shape.dtype == APMG_F32 ? 4 : 8;
  const size_t mb = es * size_t(s->off[4]), tb = es * 16 * size_t(s->shape.grids);
  if (main_m) APMG_CUDA_TRY(cudaMemcpyAsync(main_m, s->am, mb, cudaMemcpyDeviceToDevice, st));
  if (main_v) APMG_CUDA_TRY(cudaMemcpyAsync(main_v, s->av, mb, cudaMemcpyDeviceToDevice, st));
  if (tf_m) APMG_CUDA_TRY(cudaMemcpyAsync(tf_m, s->tm, tb, cudaMemcpyDeviceToDevice, st));
  if (tf_v) APMG_CUDA_TRY(cudaMemcpyAsync(tf_v, s->tv, tb, cudaMemcpyDeviceToDevice, st));
  return APMG_OK;
}

extern "C" int apmg_train_log(apmg_train_state* s, double* l_rec, double* l_density, double* lr, int64_t* stop_iteration,
                              int64_t* triggers, int64_t* n_triggers, void* stream) {
  APMG_ARG_CHECK(s != nullptr, "null state");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  TrainCtl c;
  const int64_t n = s->cfg.iterations;
  APMG_CUDA_TRY(cudaMemcpyAsync(&c, s->ctl, sizeof(c), cudaMemcpyDeviceToHost, st));
  if (l_rec) APMG_CUDA_TRY(cudaMemcpyAsync(l_rec, s->l_rec, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  if (l_density) APMG_CUDA_TRY(cudaMemcpyAsync(l_density, s->l_dens, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  if (lr) APMG_CUDA_TRY(cudaMemcpyAsync(lr, s->lr, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  if (triggers)
    APMG_CUDA_TRY(cudaMemcpyAsync(triggers, s->trig, sizeof(int64_t) * std::max<int64_t>(s->cfg.plateau_max_triggers, 1),
                                  cudaMemcpyDeviceToHost, st));
  APMG_CUDA_TRY(cudaStreamSynchronize(st));
  if (stop_iteration) *stop_iteration = c.stop_iteration;
  if (n_triggers) *n_triggers = c.n_triggers;
  return APMG_OK;
}

extern "C" int apmg_train_destroy(apmg_train_state* s) {
  if (s && s->graph) cudaGraphExecDestroy(s->graph);
  if (s && s->side) {
    cudaStreamSynchronize(s->side);
    cudaStreamDestroy(s->side);
  }
  if (s && s->ev_fork) cudaEventDestroy(s->ev_fork);
  if (s && s->ev_join) cudaEventDestroy(s->ev_join);
  if (s && s->vol_bricked && s->vol_owned) {
    cudaDeviceSynchronize();  // as cudaFree would: no launch may still read the block
    pool_free(s->vol_bricked, s->vol_bricked_bytes);
  }
  delete s;
  return APMG_OK;
}

extern "C" int apmg_host_plateau_step(double* history, int64_t* count, int64_t* triggers, int64_t window,
                                      double threshold, int64_t max_triggers, double current_ma) {
  return plateau_step_rule(history, count, triggers, window, threshold, max_triggers, current_ma);
}

extern "C" int apmg_host_transform_stop(const double* history, int64_t count, int64_t window, double threshold,
                                        int64_t hard_stop_iteration, int64_t iteration) {
  return transform_stop_rule(history, count, window, threshold, hard_stop_iteration, iteration) ? 1 : 0;
}

extern "C" double apmg_host_pairwise_sum(const double* x, int64_t n) { return ring_pairwise_sum(x, n > 0 ? n : 1, 0, n); }
