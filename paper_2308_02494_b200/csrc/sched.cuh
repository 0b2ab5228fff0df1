// Training-loop control rules shared by the device controller kernel and the
// host test hooks (same source, so the CPU tests exercise the device logic).
//   plateau_step          trainer.py:118-138
//   transform_stop_check  trainer.py:141-157
// Moving averages use numpy's pairwise summation (np.mean over a Python list
// of floats), reproduced exactly so trigger iterations match the reference.
#pragma once

#include <stdint.h>

#ifdef __CUDACC__
#define APMG_HD __host__ __device__
#else
#define APMG_HD
#endif

namespace apmg {

// numpy pairwise_sum_DOUBLE (8-way unrolled blocks of <= 128, recursive halving)
// over ring[(start + i) % cap] for i < n.
APMG_HD inline double ring_pairwise_sum(const double* ring, int64_t cap, int64_t start, int64_t n) {
  // explicit stack instead of recursion (depth <= 64)
  int64_t st_lo[64], st_n[64], st_state[64];
  double st_left[64];
  int sp = 0;
  double result = 0.0;
  st_lo[0] = start;
  st_n[0] = n;
  st_state[0] = 0;
  for (;;) {
    const int64_t lo = st_lo[sp], cnt = st_n[sp];
    double val;
    if (cnt < 8) {
      double r = 0.0;
      for (int64_t i = 0; i < cnt; ++i) r += ring[(lo + i) % cap];
      val = r;
    } else if (cnt <= 128) {
      double r[8];
      for (int j = 0; j < 8; ++j) r[j] = ring[(lo + j) % cap];
      int64_t i = 8;
      for (; i < cnt - (cnt % 8); i += 8)
        for (int j = 0; j < 8; ++j) r[j] += ring[(lo + i + j) % cap];
      double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
      for (; i < cnt; ++i) res += ring[(lo + i) % cap];
      val = res;
    } else {
      int64_t n2 = cnt / 2;
      n2 -= n2 % 8;
      // descend into the left half first
      st_state[sp] = 1;
      ++sp;
      st_lo[sp] = lo;
      st_n[sp] = n2;
      st_state[sp] = 0;
      continue;
    }
    // unwind with the value of the node at sp
    for (;;) {
      if (sp == 0) {
        result = val;
        return result;
      }
      --sp;
      const int64_t plo = st_lo[sp], pn = st_n[sp];
      int64_t n2 = pn / 2;
      n2 -= n2 % 8;
      if (st_state[sp] == 1) {  // left done: remember it, descend right
        st_left[sp] = val;
        st_state[sp] = 2;
        ++sp;
        st_lo[sp] = plo + n2;
        st_n[sp] = pn - n2;
        st_state[sp] = 0;
        break;
      }
      val = st_left[sp] + val;  // right done
    }
  }
}

// plateau_step: history is a ring of capacity window + 1 holding the most recent
// entries of PlateauState.history; *count is len(history).  Returns 0 'none',
// 1 'reduce_lr', 2 'stop'.
APMG_HD inline int plateau_step_rule(double* ring, int64_t* count, int64_t* triggers, int64_t window, double threshold,
                                     int64_t max_triggers, double current_ma) {
  const int64_t cap = window + 1;
  ring[*count % cap] = current_ma;
  *count += 1;
  if (*count <= window) return 0;
  const double ref = ring[(*count - 1 - window) % cap];
  const double aref = ref < 0 ? -ref : ref;
  const double improvement = (ref - current_ma) / (aref > 1e-12 ? aref : 1e-12);
  if (improvement >= threshold) return 0;
  *count = 0;
  *triggers += 1;
  return (*triggers >= max_triggers) ? 2 : 1;
}

// transform_stop_check over the dense density-loss history hist[0..count)
APMG_HD inline bool transform_stop_rule(const double* hist, int64_t count, int64_t window, double threshold,
                                        int64_t hard_stop_iteration, int64_t iteration) {
  if (iteration >= hard_stop_iteration) return true;
  if (count < 2 * window) return false;
  const int64_t cap = count > 0 ? count : 1;
  const double recent = ring_pairwise_sum(hist, cap, count - window, window) / double(window);
  const double previous = ring_pairwise_sum(hist, cap, count - 2 * window, window) / double(window);
  const double ap = previous < 0 ? -previous : previous;
  const double improvement = (previous - recent) / (ap > 1e-12 ? ap : 1e-12);
  return improvement < threshold;
}

}  // namespace apmg
