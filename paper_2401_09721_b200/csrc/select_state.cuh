// select_q bookkeeping shared by the single-GPU and slab filter kernels:
// Eq. (6) (filtering.py:197-222) and the FSLR outcome -> initial state.
#pragma once

#include "fgbd_internal.cuh"

namespace fgbd {

__device__ __forceinline__ double criterion(const double sy[3], const double sx[3],
                                            long long count, double sv2, int mode) {
  if (mode == FGBD_CRIT_POOLED) {
    const double ty = (sy[0] + sy[1]) + sy[2];
    const double tx = (sx[0] + sx[1]) + sx[2];
    const double lost = (ty - tx) / ((double)count * 3.0);
    return fabs(sv2 - lost);
  }
  double acc = 0.0;
#pragma unroll
  for (int c = 0; c < 3; ++c) acc += fabs(sv2 - (sy[c] - sx[c]) / (double)count);
  return acc / 3.0;
}

// Totals (count, sum_inc y^2 [3], sum_all y^2 [3]) -> FSLR outcome and the
// select_q initial state (filtering.py:237-243, 289-293).
__device__ __forceinline__ void mask_finalize(Ctl* c, const double (&t)[7], int64_t n_total, bool explicit_inc,
                              int active, int q_max, int mode, int early_exit, double sv2) {
  long long cnt = (long long)t[0];
  const bool all_ex = (cnt == 0) && !explicit_inc && active;
  c->all_excluded = all_ex;
  c->mask_all = all_ex;
  if (all_ex) {
    cnt = n_total;
    for (int k = 0; k < 3; ++k) c->sy[k] = t[4 + k];
  } else {
    for (int k = 0; k < 3; ++k) c->sy[k] = t[1 + k];
  }
  c->included = cnt;
  // select_q initial state: x = y, q = 0 (filtering.py:237-243)
  const double crit0 = cnt > 0 ? criterion(c->sy, c->sy, cnt, sv2, mode) : 0.0;
  c->q = 0;
  c->best_q = 0;
  c->best_crit = crit0;
  c->prev_crit = crit0;
  c->streak = 0;
  c->steps = 0;
  c->in_buf = BUF_Y;
  c->best_buf = BUF_Y;
  c->out_buf = BUF_A;
  c->stop = (q_max <= 0) || (crit0 == 0.0) || (cnt < 1);
  c->trace[0] = crit0;
  c->sv2 = sv2;
  c->q_max = q_max;
  c->mode = mode;
  c->early_exit = early_exit;
}

// select_q bookkeeping of one decided step (filtering.py:246-255)
struct SelState {
  int q, best_q, streak, stop, in_b, out_b, best_b;
  double best_crit, prev;
};

__device__ __forceinline__ void select_update(SelState& s, double crit, int q_max,
                                              int early_exit) {
  s.q += 1;
  if (crit < s.best_crit) {
    s.best_crit = crit;
    s.best_q = s.q;
    s.best_b = s.out_b;
  }
  s.streak = crit > s.prev ? s.streak + 1 : 0;
  s.prev = crit;
  s.stop = (early_exit && s.streak >= 3) || (s.q >= q_max) || (s.best_crit == 0.0);
  const int nin = s.out_b;
  int nout = BUF_A;  // first of A, B, Y that is neither the new input nor the best
  if (nout == nin || nout == s.best_b) nout = BUF_B;
  if (nout == nin || nout == s.best_b) nout = BUF_Y;
  s.in_b = nin;
  s.out_b = nout;
}

}  // namespace fgbd
