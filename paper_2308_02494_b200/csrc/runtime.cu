// Library runtime: thread-local error strings, launch accounting and the
// optional per-kernel CUDA-event timer used by bench.py for the roofline.
#include <stdarg.h>

#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace apmg {

static thread_local std::string g_err;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
}

std::atomic<uint64_t>& launch_counter() {
  static std::atomic<uint64_t> c{0};
  return c;
}

struct TimedLaunch {
  std::string name;
  cudaEvent_t a, b;
};

static std::mutex g_tmu;
static bool g_timing = false;
static std::vector<TimedLaunch> g_pending;
static std::map<std::string, std::pair<double, int64_t>> g_totals;

LaunchScope::LaunchScope(const char* n, cudaStream_t s) : name(n), stream(s) {
  if (!g_timing) return;
  cudaEvent_t e;
  if (cudaEventCreate(&e) != cudaSuccess) return;
  cudaEventRecord(e, s);
  start = e;
}

LaunchScope::~LaunchScope() {
  if (!start) return;
  cudaEvent_t e;
  if (cudaEventCreate(&e) != cudaSuccess) return;
  cudaEventRecord(e, stream);
  std::lock_guard<std::mutex> lk(g_tmu);
  g_pending.push_back({name, static_cast<cudaEvent_t>(start), e});
}

static void drain_pending() {
  for (auto& t : g_pending) {
    float ms = 0.f;
    cudaEventSynchronize(t.b);
    cudaEventElapsedTime(&ms, t.a, t.b);
    auto& tot = g_totals[t.name];
    tot.first += ms;
    tot.second += 1;
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  g_pending.clear();
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// Block cache for the library's own large device buffers (the bricked volume copy of a
// training session).  cudaMalloc / cudaFree of a 0.5 GiB block cost 10-200 ms each and
// cudaFree synchronises the device; sessions are created back to back (train_single,
// the decomposed trainer's per-brick sessions), so freed blocks are kept and handed to
// the next request of a similar size.  Cached blocks are released when an allocation
// fails and by apmg_release_cached().
static std::mutex g_pmu;
static std::multimap<size_t, void*> g_pool;  // size -> free block

void* pool_alloc(size_t bytes) {
  {
    std::lock_guard<std::mutex> lk(g_pmu);
    auto it = g_pool.lower_bound(bytes);
    if (it != g_pool.end() && it->first <= bytes + bytes / 4) {
      void* p = it->second;
      g_pool.erase(it);
      return p;
    }
  }
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) == cudaSuccess) return p;
  cudaGetLastError();
  release_pool();
  if (cudaMalloc(&p, bytes) == cudaSuccess) return p;
  cudaGetLastError();
  return nullptr;
}

void pool_free(void* p, size_t bytes) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_pmu);
  g_pool.emplace(bytes, p);
}

size_t pool_cached_bytes() {
  std::lock_guard<std::mutex> lk(g_pmu);
  size_t t = 0;
  for (auto& kv : g_pool) t += kv.first;
  return t;
}

void release_pool() {
  std::lock_guard<std::mutex> lk(g_pmu);
  for (auto& kv : g_pool) cudaFree(kv.second);
  g_pool.clear();
}

// Stream-ordered scratch for per-call temporaries (sweep tables, x-pair copies, SSE partials):
// allocation and release are ordered on the caller's stream, so concurrent calls on different
// streams never share a buffer.  The device's default pool keeps its memory between calls.
void* stream_alloc(size_t bytes, cudaStream_t st) {
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  });
  void* p = nullptr;
  if (cudaMallocAsync(&p, bytes, st) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}

void stream_free(void* p, cudaStream_t st) {
  if (p) cudaFreeAsync(p, st);
}

}  // namespace apmg

using namespace apmg;

extern "C" int apmg_host_register(void* ptr, size_t bytes) {
  APMG_ARG_CHECK(ptr != nullptr && bytes > 0, "null or empty host range");
  APMG_CUDA_TRY(cudaHostRegister(ptr, bytes, cudaHostRegisterDefault));
  return APMG_OK;
}

extern "C" int apmg_host_unregister(void* ptr) {
  APMG_ARG_CHECK(ptr != nullptr, "null host pointer");
  APMG_CUDA_TRY(cudaHostUnregister(ptr));
  return APMG_OK;
}

extern "C" int apmg_copy_h2d(void* dst, const void* src, size_t bytes, void* stream) {
  APMG_ARG_CHECK(dst != nullptr && src != nullptr, "null pointer");
  APMG_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, static_cast<cudaStream_t>(stream)));
  return APMG_OK;
}

extern "C" int apmg_release_cached(void) {
  release_pool();
  return APMG_OK;
}

extern "C" const char* apmg_last_error(void) { return g_err.c_str(); }
extern "C" const char* apmg_version(void) { return "apmg-b200 0.1 sm_100a"; }
extern "C" int apmg_device_sm_count(void) { return num_sms(); }
extern "C" uint64_t apmg_launch_count(void) { return launch_counter().load(); }

bool apmg::kernel_timing_on() { return g_timing; }

extern "C" int apmg_kernel_timing_enable(int on) {
  std::lock_guard<std::mutex> lk(g_tmu);
  if (!on) drain_pending();
  g_timing = on != 0;
  if (on) g_totals.clear();
  return APMG_OK;
}

extern "C" int apmg_kernel_timing_read(char* names, double* total_ms, int64_t* launches, int cap) {
  std::lock_guard<std::mutex> lk(g_tmu);
  drain_pending();
  int i = 0;
  for (auto& kv : g_totals) {
    if (i >= cap) break;
    snprintf(names + 64 * i, 64, "%s", kv.first.c_str());
    total_ms[i] = kv.second.first;
    launches[i] = kv.second.second;
    ++i;
  }
  return i;
}
