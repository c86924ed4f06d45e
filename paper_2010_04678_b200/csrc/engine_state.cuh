// Device-resident state of the fused CALS engine (csrc/engine.cu) and the
// stopping rule shared by the update kernels (engine.cu, update2.cu).
#pragma once

#include "common.cuh"
#include "internal.h"

namespace cals {

enum Status : int { kPending = 0, kActive = 1, kConverged = 2, kCap = 3, kFailed = 4 };
enum MoveKind : int { kMoveKeep = 0, kMoveRetire = 1, kMoveAdmit = 2 };

struct EngState {
  // scalars
  int order, n_models, capacity, max_slots;
  int width, n_active, queue_head, n_retired;
  int plans_done;   // number of plan() calls that did work (trace records)
  int done;
  int old_width, n_moves, move_elems;
  int max_rank;
  double tol, sqnorm;
  int max_iterations;
  long long ld;
  long long dims[kMaxOrder];
  // slots
  int* slot_model;
  int* slot_off;
  // per slot {model, rank, column offset, Gramian offset}: written by the plan
  // kernel next to slot_model / slot_off, read by the update kernel in one
  // load (no slot -> model -> rank / offset dependent round trips)
  int4* slot_info;
  // models that left the active state since the last plan (decide_model);
  // zero -> the next plan is a no-op (no retirement frees width, so no
  // admission is possible either)
  int* changed;
  // Lo-slice carry (UpdArgs::lo[1]): 1 when the column layout changed since
  // the solve kernel last wrote the next mode-0 contraction's Lo slices (set
  // by a plan that did work and at reset), 0 once that solve has written them
  int* lo_stale;
  // move plan
  int* mv_kind;
  int* mv_model;
  int* mv_src;
  int* mv_dst;
  int* mv_len;
  int* mv_pre;  // exclusive prefix of lengths
  // per model (const)
  const int* rank;
  const long long* pool_off;  // [k * order + n]
  const long long* gram_off;  // [k]
  long long gram_stride;
  // per model (state)
  int* status;
  int* iters;
  int* failed;
  int* fresh;
  int* retire_seq;
  double* f_prev;
  double* err;
  double* fit;
  unsigned long long* t_admit;
  unsigned long long* t_retire;
  double* grams;  // [order][gram_stride]
  double* pool;
  double* F[kMaxOrder];
  double* Mout;
  double* scratch;  // per-block pinv scratch
  // trace
  int tr_cap;
  int* tr_width;
  int* tr_active;
  unsigned long long* tr_time;
  volatile int* host_done;
  // line search (als.py:127-144, driver.py:250-259,272-273): snapshots S of
  // the previous iterate, candidates C, their Gramians, per-model flags
  int ls_enabled;
  double ls_alpha;  // <= 0: alpha = iteration^(1/3)
  double* S[kMaxOrder];
  double* Cb[kMaxOrder];
  double* cgrams;
  int* has_snap;
  int* ls_act;
  double* e_tmp;
  // non-negative updates (als.py:185-278): per model, mode and factor row
  // the active-set bitmask carried between iterations
  int nonneg;
  unsigned* nnls_state;
  const long long* nnls_off;  // [k * order + n]
  int* nnls_warn;             // a row hit the active-set iteration cap
  // split update (update2.cuh): per-model solve arrival counters and flags
  int* arrive;
  int* solbad;
};

// Per-model scalars of the stopping rule, loadable ahead of time (all
// loads independent) so the decision itself is loads-free.
struct DecideIn {
  int it;        // iteration count after this iteration's increment
  int failed;
  double f_prev;
  double tol, sqnorm;
  int max_iterations;
};

// Stopping rule for model k with squared error e (driver.py:260-273); the
// caller has already incremented iters[k].  Thread 0 only.
__device__ inline void decide_model_with(EngState* st, int k, double e, const DecideIn& d) {
  if (d.failed) {
    st->err[k] = nan("");
    st->fit[k] = -INFINITY;
    st->status[k] = kFailed;
    atomicAdd(st->changed, 1);
    return;
  }
  if (!isfinite(e)) {
    st->err[k] = e;
    st->fit[k] = -INFINITY;
    st->status[k] = kFailed;
    atomicAdd(st->changed, 1);
    return;
  }
  const double f = 1.0 - sqrt(e) / sqrt(d.sqnorm);
  st->err[k] = e;
  st->fit[k] = f;
  if (d.tol > 0.0 && f - d.f_prev < d.tol) {
    st->status[k] = kConverged;
    atomicAdd(st->changed, 1);
  } else if (d.it >= d.max_iterations) {
    st->status[k] = kCap;
    atomicAdd(st->changed, 1);
  } else {
    st->f_prev[k] = f;
  }
}

__device__ inline void decide_model(EngState* st, int k, double e) {
  DecideIn d;
  d.it = st->iters[k];
  d.failed = st->failed[k];
  d.f_prev = st->f_prev[k];
  d.tol = st->tol;
  d.sqnorm = st->sqnorm;
  d.max_iterations = st->max_iterations;
  decide_model_with(st, k, e, d);
}

}  // namespace cals
