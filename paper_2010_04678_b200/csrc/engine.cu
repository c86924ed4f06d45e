// Device-resident CALS driver (Algorithm 4 of arXiv 2010.04678).
//
// Restates pkg/src/cals/driver.py:185-307 (`_run_cals`) with every piece of
// per-iteration state in HBM:
//   * factor multi-matrices, one row-major [I_n][ld] buffer per mode (the
//     reference keeps Fortran (I_n, R*) buffers, multimatrix.py:33-120);
//   * per-model Gramians, status, iteration count, f_prev, error, fit;
//   * the slot layout (registry order) and the FIFO admission queue.
// One driver iteration is a fixed kernel sequence captured once in a CUDA
// graph:  for n in modes: [fused MTTKRP(n) -> split reduce -> update(n)]
// (fit fused into update(N-1)), then plan (retire / compact / admit, trace)
// and move (retire copy-out, compaction, admission copy-in).  The host only
// replays the graph and polls a mapped "done" flag; no per-iteration host
// round trip.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <chrono>
#include <cstring>
#include <numeric>
#include <vector>

#include "internal.h"
#include "mttkrp.cuh"
#include "update.cuh"
#include "nnls.cuh"
#include "engine_state.cuh"
#include "update2.cuh"

namespace cals {
constexpr int kNnlsWs = kNnlsP * 32 + 32 + 32 * 32;  // per-warp NNLS scratch (doubles)
}

namespace cals {

// ------------------------------------------------------------------ update --
// RB > 0: fast path (every rank <= RB, rows in registers, chunked Gram);
// RB == 0: generic path (block Cholesky / row solves / Jacobi pinv) for ranks
// up to kMaxRank; up to kSmemRankMax the R x R matrix lives in shared memory,
// above it in the block's global scratch slice (L2-resident).  Same
// reference semantics.
#ifdef CALS_UPD_PROFILE
__device__ long long g_upd_prof[3][4096][13];
#define UPD_STAMP(i) \
  if (threadIdx.x == 32) ustamp[i] = clock64();
#else
#define UPD_STAMP(i)
#endif
template <int RB>
__global__ void __launch_bounds__(kUpdThreads, 2) engine_update_kernel(
    EngState* st_g, const int4* __restrict__ slot_info, int n, int nthr) {
  extern __shared__ __align__(16) double dsm[];
  __shared__ int flag;
  __shared__ double red[kUpdThreads];
  // The engine state (pointers and scalars, fixed for this launch) is read
  // through a shared-memory copy: every st-> access in the per-model chain
  // is then one smem load instead of a dependent global round trip.  Writes
  // go through the copied pointers into the global arrays.
  __shared__ __align__(16) EngState sst;
#ifdef CALS_UPD_PROFILE
  __shared__ long long ustamp[10];
  const long long t_entry = (long long)globaltimer_ns();
  const long long c_entry = clock64();
#endif
  // this block's first slot record is loaded alongside the state copy
  // (blockIdx.x < max_slots: always in bounds; used only if the slot is active)
  const int4 si_first = slot_info[blockIdx.x];
  for (int i = threadIdx.x; i < int(sizeof(EngState) / 4); i += blockDim.x)
    reinterpret_cast<int*>(&sst)[i] = reinterpret_cast<const int*>(st_g)[i];
  __syncthreads();
  UPD_STAMP(0)
  EngState* const st = &sst;
  const int N = st->order;
  const int Rmax = st->max_rank;
  const bool big = Rmax > kSmemRankMax;
  double* V = st->scratch + (long long)blockIdx.x * upd_scratch_doubles(Rmax);
  double* Hsave = V + Rmax * Rmax;
  double* lam = Hsave + Rmax * Rmax;
  double* H = big ? lam + Rmax : dsm;     // Rmax^2
  double* X = big ? dsm : H + Rmax * Rmax;  // generic: Rmax * nthr; fast: kUpdThreads * (RB + 1)
  const int rows = (int)st->dims[n];
  const long long ld = st->ld;
  const int n_active = st->n_active;

  for (int slot = blockIdx.x; slot < n_active; slot += gridDim.x) {
    const int4 si = slot == (int)blockIdx.x ? si_first : slot_info[slot];
    const int k = si.x;
    const int R = si.y;
    const int off = si.z;
    const long long go = si.w;
    auto gram = [&](int i) { return st->grams + i * st->gram_stride + go; };
    UPD_STAMP(1)

    if (n == 0 && st->fresh[k]) {
      // Gramians of the admitted starting point (driver.py:203-205)
      for (int i = 1; i < N; ++i) {
        if constexpr (RB > 0)
          block_gram_fast<RB>(st->F[i] + off, ld, (int)st->dims[i], R, X, gram(i));
        else
          block_gram(st->F[i], ld, off, (int)st->dims[i], R, gram(i));
      }
      if (st->nonneg) {  // NnlsState(t.dims, rank): nothing pinned (driver.py:206)
        for (int i = 0; i < N; ++i) {
          unsigned* sp = st->nnls_state + st->nnls_off[(long long)k * N + i];
          for (long long r = threadIdx.x; r < st->dims[i]; r += blockDim.x) sp[r] = 0u;
        }
        if (threadIdx.x == 0) st->nnls_warn[k] = 0;
      }
      __syncthreads();
      if (threadIdx.x == 0) st->fresh[k] = 0;
    }
    bool updated = false;
    double inner = 0.0;
    bool have_inner = false;
    if (!st->failed[k]) {
      int bad = 0;
      for (int idx = threadIdx.x; idx < R * R; idx += blockDim.x) {
        double h = 1.0;
        bool first = true;
        for (int i = 0; i < N; ++i) {
          if (i == n) continue;
          const double g = gram(i)[idx];
          h = first ? g : h * g;
          first = false;
        }
        H[idx] = h;
        Hsave[idx] = h;
        bad |= !isfinite(h);
      }
      const double* Mb = st->Mout + off;
      __shared__ double inv_diag[kFastR];
      bool chol_ok = false;
      if constexpr (RB > 0) {
        // warp 0 factors H while the other warps check the whole M block and
        // stage its first chunk of rows into X (the reference checks before
        // touching anything, als.py:84-85; a NaN pivot is caught below too)
        __syncthreads();
        UPD_STAMP(2)
        if (threadIdx.x < 32) {
          warp_cholesky_fast_nosync<RB>(H, R, inv_diag, &flag);
        } else {
          const int P = fast_pitch(R);
          const int nt = blockDim.x - 32;
          const int c0 = min(rows, kUpdThreads);
          bad |= stage_block(Mb, ld, c0, R, P, X, threadIdx.x - 32, nt);
          if (rows > c0)
            bad |= stage_block(Mb + (long long)c0 * ld, ld, rows - c0, R, P, nullptr,
                               threadIdx.x - 32, nt);
        }
      } else {
        for (int i = threadIdx.x; i < rows; i += blockDim.x) {
          const double* mrow = Mb + (long long)i * ld;
          for (int a = 0; a < R; ++a) bad |= !isfinite(mrow[a]);
        }
      }
      const int any_bad = __syncthreads_or(bad);
      UPD_STAMP(3)
      if (any_bad) {
        // non-finite input: the reference raises ValueError -> FAILED (als.py:84-85)
        if (threadIdx.x == 0) st->failed[k] = 1;
        __syncthreads();
      } else {
        bool done = false;
        if (st->nonneg) {
          // non-negative update (driver.py:226-227 -> nnls_update): one warp
          // per factor row, warm-started active sets kept per row
          for (int idx = threadIdx.x; idx < R * R; idx += blockDim.x) H[idx] = Hsave[idx];
          __syncthreads();
          const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
          double* Ws = X + warp * kNnlsWs;
          unsigned* state = st->nnls_state + st->nnls_off[(long long)k * N + n];
          for (int i = warp; i < rows; i += blockDim.x >> 5) {
            const double f = lane < R ? Mb[(long long)i * ld + lane] : 0.0;
            unsigned act = state[i];
            bool conv = true;
            const double x = nnls_row(H, R, f, &act, &conv, Ws);
            if (lane < R) st->F[n][(long long)i * ld + off + lane] = x;
            if (lane == 0) {
              state[i] = act;
              if (!conv) st->nnls_warn[k] = 1;
            }
          }
          __syncthreads();
          block_gram_fast<(RB > 0 ? RB : kFastR)>(st->F[n] + off, ld, rows, R, X, gram(n));
          done = true;
        }
        if constexpr (RB > 0) {
          chol_ok = !done && flag != 0;
          if (chol_ok) {
            done = block_solve_gram_fast<RB>(H, inv_diag, R, Mb, ld, rows, st->F[n] + off, ld, X,
                                         gram(n), n == N - 1, &inner, red, true
#ifdef CALS_UPD_PROFILE
                                         , ustamp + 6
#endif
            );
            have_inner = done && n == N - 1;
          }
          UPD_STAMP(4)
        }
        if (!done) {
          for (int idx = threadIdx.x; idx < R * R; idx += blockDim.x) H[idx] = Hsave[idx];
          __syncthreads();
          block_update(H, Hsave, V, lam, X, nthr, R, Mb, ld, rows, st->F[n] + off, ld, &flag);
          block_gram(st->F[n], ld, off, rows, R, gram(n));
        }
        updated = true;
      }
      __syncthreads();
    }
    UPD_STAMP(5)
    if (n == N - 1) {
      // fast error / fit / stopping rule (driver.py:241-273, als.py:99-124)
      double msq = 0.0;
      if (updated) {
        if (!have_inner) {
          double part = 0.0;
          for (long long e = threadIdx.x; e < (long long)rows * R; e += blockDim.x) {
            const long long i = e / R;
            const int r = int(e % R);
            part = fma(st->F[n][i * ld + off + r], st->Mout[i * ld + off + r], part);
          }
          inner = block_sum(part, red);
        }
        double mpart = 0.0;
        for (int idx = threadIdx.x; idx < R * R; idx += blockDim.x) {
          double h = gram(0)[idx];
          for (int i = 1; i < N; ++i) h *= gram(i)[idx];
          mpart += h;
        }
        msq = block_sum(mpart, red);
      }
      if (threadIdx.x == 0) {
        ++st->iters[k];
        double e = st->sqnorm + msq - 2.0 * inner;
        e = e > 0.0 ? e : 0.0;  // als.py:114-115 (NaN clamps to 0 as there)
        if (st->ls_enabled)
          st->e_tmp[k] = e;  // decided after the line-search candidate (ls_finish)
        else
          decide_model(st, k, e);
      }
      __syncthreads();
    }
#ifdef CALS_UPD_PROFILE
    if (threadIdx.x == 0 && slot < 4096 && n < 3) {
      g_upd_prof[n][slot][0] = t_entry;
      g_upd_prof[n][slot][1] = (long long)globaltimer_ns();
      g_upd_prof[n][slot][2] = clock64() - c_entry;
      g_upd_prof[n][slot][3] = R;
      for (int i = 0; i < 9; ++i) g_upd_prof[n][slot][4 + i] = ustamp[i] - c_entry;
    }
#endif
  }
}

// ------------------------------------------------------------- line search --
// Candidate point prev + alpha (curr - prev) for every model holding a
// snapshot (extrapolate_factors, als.py:137-138: evaluated as
// p + alpha * (c - p) with three roundings, no FMA contraction) and its
// Gramians; models without a snapshot or with a non-finite error skip.
__global__ void __launch_bounds__(kUpdThreads) ls_candidate_kernel(EngState* st) {
  extern __shared__ __align__(16) double dsm[];
  const int N = st->order;
  const long long ld = st->ld;
  for (int slot = blockIdx.x; slot < st->n_active; slot += gridDim.x) {
    const int k = st->slot_model[slot];
    const int R = st->rank[k];
    const int off = st->slot_off[slot];
    const bool act = !st->failed[k] && st->has_snap[k] && isfinite(st->e_tmp[k]);
    if (threadIdx.x == 0) st->ls_act[k] = act ? 1 : 0;
    if (!act) continue;
    const double alpha =
        st->ls_alpha > 0.0 ? st->ls_alpha : pow((double)st->iters[k], 1.0 / 3.0);
    for (int n = 0; n < N; ++n) {
      const int rows = (int)st->dims[n];
      for (long long e = threadIdx.x; e < (long long)rows * R; e += blockDim.x) {
        const long long i = e / R;
        const long long at = i * ld + off + (e - i * R);
        const double p = st->S[n][at], c = st->F[n][at];
        st->Cb[n][at] = __dadd_rn(p, __dmul_rn(alpha, __dsub_rn(c, p)));
      }
    }
    __syncthreads();
    for (int n = 0; n < N; ++n) {
      double* G = st->cgrams + n * st->gram_stride + st->gram_off[k];
      if (R <= kFastR)
        block_gram_fast(st->Cb[n] + off, ld, (int)st->dims[n], R, dsm, G);
      else
        block_gram(st->Cb[n], ld, off, (int)st->dims[n], R, G);
    }
    __syncthreads();
  }
}

// Candidate error from the fresh last-mode MTTKRP of the candidates (Mout),
// keep the better point (driver.py:255-259), then the stopping rule and the
// snapshot of a continuing model (driver.py:271-273).
__global__ void __launch_bounds__(kUpdThreads) ls_finish_kernel(EngState* st) {
  __shared__ double red[kUpdThreads];
  __shared__ int accept;
  const int N = st->order;
  const long long ld = st->ld;
  const int n = N - 1;
  for (int slot = blockIdx.x; slot < st->n_active; slot += gridDim.x) {
    const int k = st->slot_model[slot];
    const int R = st->rank[k];
    const int off = st->slot_off[slot];
    const long long go = st->gram_off[k];
    double e = st->e_tmp[k];
    if (st->ls_act[k]) {
      const int rows = (int)st->dims[n];
      double part = 0.0;
      for (long long el = threadIdx.x; el < (long long)rows * R; el += blockDim.x) {
        const long long i = el / R;
        const long long at = i * ld + off + (el - i * R);
        part = fma(st->Cb[n][at], st->Mout[at], part);
      }
      const double inner = block_sum(part, red);
      double mp = 0.0;
      for (int idx = threadIdx.x; idx < R * R; idx += blockDim.x) {
        double h = st->cgrams[go + idx];
        for (int i = 1; i < N; ++i) h *= st->cgrams[i * st->gram_stride + go + idx];
        mp += h;
      }
      const double msq = block_sum(mp, red);
      double ec = st->sqnorm + msq - 2.0 * inner;
      ec = ec > 0.0 ? ec : 0.0;
      if (threadIdx.x == 0) accept = ec < e ? 1 : 0;
      __syncthreads();
      if (accept) {
        e = ec;
        for (int m = 0; m < N; ++m) {
          const int rm = (int)st->dims[m];
          for (long long el = threadIdx.x; el < (long long)rm * R; el += blockDim.x) {
            const long long i = el / R;
            const long long at = i * ld + off + (el - i * R);
            st->F[m][at] = st->Cb[m][at];
          }
          for (int idx = threadIdx.x; idx < R * R; idx += blockDim.x)
            st->grams[m * st->gram_stride + go + idx] = st->cgrams[m * st->gram_stride + go + idx];
        }
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) decide_model(st, k, e);
    __syncthreads();
    if (st->status[k] == kActive) {
      // continuing: snapshot the (possibly extrapolated) iterate
      for (int m = 0; m < N; ++m) {
        const int rm = (int)st->dims[m];
        for (long long el = threadIdx.x; el < (long long)rm * R; el += blockDim.x) {
          const long long i = el / R;
          const long long at = i * ld + off + (el - i * R);
          st->S[m][at] = st->F[m][at];
        }
      }
      if (threadIdx.x == 0) st->has_snap[k] = 1;
    }
    __syncthreads();
  }
}

using UpdateKernel = void (*)(EngState*, const int4*, int, int);
static UpdateKernel update_kernel_for(int max_rank, int* rb) {
  // rank buckets: the per-thread register arrays (Cholesky column, solved
  // row, Gram pairs) are sized to the largest rank of the batch
  if (max_rank <= 8) { *rb = 8; return engine_update_kernel<8>; }
  if (max_rank <= 16) { *rb = 16; return engine_update_kernel<16>; }
  if (max_rank <= 24) { *rb = 24; return engine_update_kernel<24>; }
  if (max_rank <= kFastR) { *rb = kFastR; return engine_update_kernel<kFastR>; }
  *rb = 0;
  return engine_update_kernel<0>;
}

// -------------------------------------------------------------------- plan --
// One block: retire (registry order), compact survivors, admit FIFO with
// head-of-line blocking (driver.py:198-208, 274-276; multimatrix.py:103-158).
// block-wide inclusive scan of one int per thread (blockDim.x = kPlanThreads)
constexpr int kPlanThreads = 1024;
__device__ __forceinline__ int plan_scan(int v, int* wtot, int* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) wtot[w] = incl;
  __syncthreads();
  if (w == 0) {
    int t = wtot[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += u;
    }
    wtot[lane] = t;  // inclusive over warps
  }
  __syncthreads();
  const int r = incl + (w > 0 ? wtot[w - 1] : 0);
  *total = wtot[31];
  __syncthreads();
  return r;
}

// Retire / compact / admit (driver.py:199-208, 274-276; multimatrix.py:97-158)
// for one driver iteration.  One block of kPlanThreads: every slot's model,
// status, rank and offset are loaded in parallel, the prefix sums (kept
// widths, move lengths, retirement order) are block scans, and only the FIFO
// admission with head-of-line blocking runs on one thread.
__global__ void __launch_bounds__(kPlanThreads, 1) engine_plan_kernel(EngState* st) {
  griddep_wait();  // launched with PDL (launch_dep): predecessors complete
  if (st->done) return;
  __shared__ int wtot[32];
  __shared__ int s_new_w, s_new_n, s_retired, s_moves, s_pre;
  const unsigned long long now = globaltimer_ns();
  if (st->plans_done > 0 && *st->changed == 0) {
    // nothing retired: same slots, no moves, no admission possible; only the
    // trace record (driver.py:278-284) and the plan count
    if (threadIdx.x == 0) {
      const int rec = st->plans_done;
      st->old_width = st->width;
      st->move_elems = 0;
      st->n_moves = 0;
      if (rec < st->tr_cap) {
        st->tr_width[rec] = st->width;
        st->tr_active[rec] = st->n_active;
        st->tr_time[rec] = now;
      }
      st->plans_done = rec + 1;
    }
    return;
  }
  const int n_old = st->n_active;
  if (threadIdx.x == 0) {
    s_new_w = 0;
    s_new_n = 0;
    s_retired = st->n_retired;
    s_moves = 0;
    s_pre = 0;
  }
  __syncthreads();
  for (int base = 0; base < n_old; base += kPlanThreads) {
    const int s = base + threadIdx.x;
    const bool valid = s < n_old;
    const int k = valid ? st->slot_model[s] : 0;
    const int src = valid ? st->slot_off[s] : 0;
    const int rank_k = valid ? st->rank[k] : 0;
    const int gram_k = valid ? (int)st->gram_off[k] : 0;
    const bool retiring = valid && st->status[k] != kActive;
    const bool keep = valid && !retiring;
    const int new_w = s_new_w, new_n = s_new_n, retired = s_retired, moves = s_moves,
              pre = s_pre;
    __syncthreads();  // everyone has read the carries (and its slot, compacted below)
    const int rk = keep ? rank_k : 0;
    int tw, tk, tr, tm;
    const int incl = plan_scan(rk, wtot, &tw);
    const int kidx = plan_scan(keep ? 1 : 0, wtot, &tk) - (keep ? 1 : 0);
    const int ridx = plan_scan(retiring ? 1 : 0, wtot, &tr) - (retiring ? 1 : 0);
    const int dst_keep = new_w + incl - rk;
    const int ml = retiring ? rank_k : (keep && dst_keep != src ? rk : 0);
    const int mincl = plan_scan(ml, wtot, &tm);
    if (valid) {
      const int mi = moves + (s - base);  // every valid slot is retiring or kept
      st->mv_pre[mi] = pre + mincl - ml;
      st->mv_model[mi] = k;
      st->mv_src[mi] = src;
      if (retiring) {
        st->retire_seq[k] = retired + ridx;
        st->t_retire[k] = now;
        st->mv_kind[mi] = kMoveRetire;
        st->mv_dst[mi] = 0;
        st->mv_len[mi] = rank_k;
      } else {
        st->mv_kind[mi] = kMoveKeep;
        st->mv_dst[mi] = dst_keep;
        st->mv_len[mi] = dst_keep != src ? rk : 0;
        // slot arrays are compacted in place: new index <= s, and every slot
        // of this chunk was read before the barrier above
        st->slot_model[new_n + kidx] = k;
        st->slot_off[new_n + kidx] = dst_keep;
        st->slot_info[new_n + kidx] = make_int4(k, rank_k, dst_keep, gram_k);
      }
    }
    if (threadIdx.x == 0) {
      s_new_w = new_w + tw;
      s_new_n = new_n + tk;
      s_retired = retired + tr;
      s_moves = moves + min(kPlanThreads, n_old - base);
      s_pre = pre + tm;
    }
    __syncthreads();
  }
  // FIFO admission with head-of-line blocking (driver.py:199-208,
  // multimatrix.py:143-158), kPlanThreads queued models per round: the
  // admitted models are the prefix whose rank prefix sum still fits, so a
  // block scan places them all at once (same slots, offsets and move list as
  // admitting one at a time).
  __shared__ int s_head, s_more;
  if (threadIdx.x == 0) s_head = st->queue_head;
  __syncthreads();
  for (;;) {
    const int head = s_head, new_w = s_new_w, new_n = s_new_n, moves = s_moves, pre = s_pre;
    if (head >= st->n_models) break;  // block-uniform
    const int k = head + threadIdx.x;
    const bool valid = k < st->n_models;
    const int rk = valid ? st->rank[k] : 0;
    int tot_r, n_adm;
    const int incl = plan_scan(rk, wtot, &tot_r);
    const bool adm = valid && (long long)new_w + incl <= (long long)st->capacity;
    plan_scan(adm ? 1 : 0, wtot, &n_adm);
    if (adm) {
      const int off = new_w + incl - rk;  // threadIdx.x = index in the admitted prefix
      st->status[k] = kActive;
      st->fresh[k] = 1;
      if (st->has_snap) st->has_snap[k] = 0;
      st->t_admit[k] = now;
      st->slot_model[new_n + threadIdx.x] = k;
      st->slot_off[new_n + threadIdx.x] = off;
      st->slot_info[new_n + threadIdx.x] = make_int4(k, rk, off, (int)st->gram_off[k]);
      const int mi = moves + threadIdx.x;
      st->mv_kind[mi] = kMoveAdmit;
      st->mv_model[mi] = k;
      st->mv_src[mi] = 0;
      st->mv_dst[mi] = off;
      st->mv_len[mi] = rk;
      st->mv_pre[mi] = pre + incl - rk;
      if ((int)threadIdx.x == n_adm - 1) {  // last admitted: carries
        s_new_w = new_w + incl;
        s_pre = pre + incl;
      }
    }
    if (threadIdx.x == 0) {
      s_head = head + n_adm;
      s_new_n = new_n + n_adm;
      s_moves = moves + n_adm;
      s_more = n_adm == kPlanThreads;
    }
    __syncthreads();
    if (!s_more) break;
  }
  if (threadIdx.x == 0) {
    const int new_w = s_new_w, new_n = s_new_n, moves = s_moves, pre = s_pre, head = s_head;
    st->old_width = st->width;
    st->move_elems = pre;
    st->n_moves = moves;
    st->queue_head = head;
    st->n_active = new_n;
    st->width = new_w;
    st->n_retired = s_retired;
    const int rec = st->plans_done;
    if (rec < st->tr_cap) {
      st->tr_width[rec] = new_w;
      st->tr_active[rec] = new_n;
      st->tr_time[rec] = now;
    }
    st->plans_done = rec + 1;
    *st->changed = 0;
    *st->lo_stale = 1;  // columns may have moved: carried Lo slices are stale
    if (new_n == 0 && head >= st->n_models) {
      st->done = 1;
      st->host_done[1] = rec + 1;  // plan count, read by the host without a copy
      __threadfence_system();
      st->host_done[0] = 1;
      __threadfence_system();
    }
  }
}

// -------------------------------------------------------------------- move --
// One block per (mode, row): snapshot the old active row, then apply the move
// list -> no in-place hazards.
__global__ void engine_move_kernel(EngState* st) {
  griddep_wait();  // launched with PDL (launch_dep): predecessors complete
  const int total = st->move_elems;
  if (total == 0) return;
  extern __shared__ __align__(16) double row[];
  const int N = st->order;
  long long rows_f = 0;
  for (int n = 0; n < N; ++n) rows_f += st->dims[n];
  // line search: the snapshot rows travel with the factor rows (KEEP only)
  const long long rows_total = st->ls_enabled ? 2 * rows_f : rows_f;
  const int ow = st->old_width;
  const int nm = st->n_moves;
  for (long long gr = blockIdx.x; gr < rows_total; gr += gridDim.x) {
    const bool snap = gr >= rows_f;
    int n = 0;
    long long i = snap ? gr - rows_f : gr;
    while (i >= st->dims[n]) {
      i -= st->dims[n];
      ++n;
    }
    double* F = (snap ? st->S[n] : st->F[n]) + i * st->ld;
    for (int c = threadIdx.x; c < ow; c += blockDim.x) row[c] = F[c];
    __syncthreads();
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
      int lo = 0, hi = nm - 1;  // last move with mv_pre <= e
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (st->mv_pre[mid] <= e) lo = mid; else hi = mid - 1;
      }
      const int r = e - st->mv_pre[lo];
      const int k = st->mv_model[lo];
      const long long po = st->pool_off[(long long)k * N + n] + r * st->dims[n] + i;
      if (snap && st->mv_kind[lo] != kMoveKeep) continue;
      switch (st->mv_kind[lo]) {
        case kMoveKeep: F[st->mv_dst[lo] + r] = row[st->mv_src[lo] + r]; break;
        case kMoveRetire: st->pool[po] = row[st->mv_src[lo] + r]; break;
        default: F[st->mv_dst[lo] + r] = st->pool[po]; break;
      }
    }
    __syncthreads();
  }
}

// ----------------------------------------------------- standalone update --
// update_factor(m, h) for one block (als.py:74-96): rows x R, row-major.
__global__ void __launch_bounds__(kUpdThreads) standalone_update_kernel(
    const double* Mb, long long ldm, int rows, int R, const double* Hin, double* A, long long lda,
    double* scratch, int nthr, int* status) {
  extern __shared__ __align__(16) double dsm[];
  __shared__ int flag;
  // scratch: V (R^2), Hsave (R^2), lam (R), and H (R^2) above kSmemRankMax
  const bool big = R > kSmemRankMax;
  double* H = big ? scratch + 2 * R * R + R : dsm;
  double* X = big ? dsm : H + R * R;
  for (int idx = threadIdx.x; idx < R * R; idx += blockDim.x) H[idx] = Hin[idx];
  __syncthreads();
  const bool ok = block_update(H, scratch + R * R, scratch, scratch + 2 * R * R, X, nthr, R, Mb,
                               ldm, rows, A, lda, &flag);
  if (threadIdx.x == 0) *status = ok ? 0 : 1;
}

// ------------------------------------------------------------------- lambdas --
// lambda_r = prod_n ||A_n[:, r]|| of every retired model (pool layout).
__global__ void lambdas_kernel(const EngState* st, const long long* lam_off, double* lam) {
  const int N = st->order;
  for (int k = blockIdx.x; k < st->n_models; k += gridDim.x) {
    const int R = st->rank[k];
    for (int r = threadIdx.x; r < R; r += blockDim.x) {
      double prod = 1.0;
      for (int n = 0; n < N; ++n) {
        const double* P = st->pool + st->pool_off[(long long)k * N + n];
        double s = 0.0;
        const double* col = P + r * st->dims[n];
        for (long long i = 0; i < st->dims[n]; ++i) s = fma(col[i], col[i], s);
        prod *= sqrt(s);
      }
      lam[lam_off[k] + r] = prod;
    }
  }
}

// ============================================================== host side ==

static int pick_nthr(int R) {
  int nthr = kUpdThreads;
  while (nthr > 32 && (long long)R * nthr * 8 > 96 * 1024) nthr -= 32;
  return nthr;
}

enum Tree : int { kTreeNone = 0, kTreeY = 1, kTreeZ = 2 };

struct Engine {
  Tensor* t = nullptr;
  int device = 0;  // CUDA device of every allocation below (the tensor's)
  unsigned long long tensor_uid = 0;
  int order = 0, n_models = 0, capacity = 0, max_slots = 0, max_rank = 0;
  long long ld = 0;
  std::vector<int> ranks;
  std::vector<long long> pool_off, gram_off, lam_off;
  long long pool_elems = 0, gram_stride = 0, lam_elems = 0;
  // device allocations
  EngState* d_st = nullptr;
  EngState h_st{};
  void* d_block = nullptr;  // one arena for everything else
  double* d_lam = nullptr;
  long long* d_lam_off = nullptr;
  size_t ws_bytes = 0;
  double* d_ws = nullptr;
  int* h_done = nullptr;  // mapped pinned: [0] done flag, [1] plans at completion
  EngState* h_st_pinned = nullptr;  // page-locked staging of the state upload
  cudaEvent_t st_upload_ev = nullptr;
  char* h_results = nullptr;  // pinned staging of the per-model results
  size_t h_results_bytes = 0;
  int* d_done_alias = nullptr;
  int variants[kMaxOrder];
  // dimension tree (order 3): share one tensor-core contraction between two modes
  int tree = 0;
  ModePlan tree_plan;
  int tree_variant = 0;
  double* d_partial = nullptr;
  double* d_ones = nullptr;
  void* d_ls = nullptr;  // line-search buffers (allocated on first enable)
  void* d_nnls = nullptr;  // NNLS active sets (allocated on first enable)
  size_t ls_smem = 0;
  int upd_grid = 0, upd_nthr = 0, upd_rb = 0;
  UpdateKernel upd_kernel = nullptr;
  size_t upd_smem = 0, move_smem = 0;
  // split update (update2.cuh): ranks <= 32, Cholesky / pinv updates.  prep(n)
  // runs on `side`, forked after the previous mode's solve and joined before
  // solve(n), i.e. concurrently with the fused MTTKRP of mode n.
  bool split = false;
  UpdArgs ua{};
  int lo_target = -1;  // mode whose contraction takes its Lo slices from solve(0)
  bool lo_carry = false;  // mode 0's Lo slices carried over from the previous iteration
  PrepKernel prep_kernel = nullptr;
  SolveKernel solve_kernel = nullptr, solve_last_kernel = nullptr;
  size_t solve_smem = 0;
  int nch[kMaxOrder] = {0};
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork[kMaxOrder] = {nullptr}, ev_join[kMaxOrder] = {nullptr};
  int move_grid = 0;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  bool graph_stale = false;  // tensor re-bound since the capture
  cudaStream_t cap_stream = nullptr;
  int trace_cap = 0;
  int last_iterations = 0;
  // kernel launches of the last engine_run: kernel nodes of the captured
  // iteration graph x graph launches + the kernels launched directly
  int graph_kernels = 0;
  long long last_launches = 0;
  // byte offset of the dimension-tree contraction's workspace in d_ws: past
  // every plain plan's (setup_tree)
  size_t tree_base = 0;
};

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Kernel attributes are process-global: several engines (different r_star,
// ranks) share the kernels, so the dynamic shared-memory limit only ever
// grows -- a cached engine must never find it lowered by a younger one.
static cudaError_t raise_smem_limit(const void* func, size_t bytes) {
  static std::mutex mu;
  static std::map<const void*, size_t> cur;
  std::lock_guard<std::mutex> lk(mu);
  size_t& have = cur[func];
  if (bytes <= have) return cudaSuccess;
  const cudaError_t e =
      cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}


// the tree contraction's split partials sit at the start of the engine
// workspace, its Ozaki Lo slices after them
static char* tree_ws(Engine* e) { return reinterpret_cast<char*>(e->d_ws) + e->tree_base; }

static size_t tree_ws_offset(const ModePlan& p, long long ld) {
  return align_up(size_t(p.S) * size_t(p.M) * size_t(ld) * 8, 256);
}

// Ozaki X slices for every view this engine contracts (built once per tensor,
// before any graph capture).
static int engine_prepare_slices(Engine* e, cudaStream_t stream, bool validate = true) {
  Tensor& t = *e->t;
  const int N = e->order;
  for (int n = 0; n < N; ++n) {
    const bool used = e->tree == kTreeNone || n == N - 1 || (e->tree == kTreeZ && n == 0);
    if (!used) continue;
    const int rc = ozaki_prepare(t, t.plans[n], n, stream, validate);
    if (rc) return rc;
  }
  if (e->tree == kTreeY) return ozaki_prepare(t, e->tree_plan, 100, stream, validate);
  if (e->tree == kTreeZ) return ozaki_prepare(t, e->tree_plan, 1, stream, validate);
  return kOk;
}

// Dimension tree for 3-way tensors (ALS order 0,1,2):
//   Y-tree: Y = X x_3 A2 is shared by modes 0 and 1 (A2 is not updated
//           between them); mode 2 is a full fused MTTKRP.
//   Z-tree: Z = X x_1 A0(new) is shared by modes 1 and 2 (A0 was updated
//           before both); mode 0 is a full fused MTTKRP.
// Two tensor-core contractions per iteration instead of three; the smaller
// partial (I0*I1 vs I1*I2 rows) is chosen.  CALS_TREE=0|1|2 overrides.
static int setup_tree(Engine* e) {
  Tensor& t = *e->t;
  e->tree = kTreeNone;
  if (t.order != 3) return kOk;
  const long long yrows = t.i0p * t.dims[1], zrows = t.dims[1] * t.dims[2];
  int choice = yrows <= zrows ? kTreeY : kTreeZ;
  if (const char* env = getenv("CALS_TREE")) choice = atoi(env);
  if (choice != kTreeY && choice != kTreeZ) return kOk;
  const long long rows = choice == kTreeY ? yrows : zrows;
  const size_t bytes = size_t(rows) * size_t(e->ld) * 8;
  size_t free_b = 0, total_b = 0;
  CALS_CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
  if (bytes > free_b / 2) return kOk;  // not worth starving the allocator
  ModePlan& p = e->tree_plan;
  if (choice == kTreeY) {
    // mode 0 as view (m = i, q = j, p = k): the tensor cores contract k, so
    // each per-slab product is Y[i, j, :] -- written once as a side output
    // while the same kernel scales by A1[j] and accumulates M0.
    p = t.plans[0];
    p.role = kRoleFirstQP;
    p.Dp = t.dims[2];
    p.Dq = t.dims[1];
    p.S = plan_splits(p);
    p.lo_modes = {2};
    p.hi_modes = {1};
  } else {
    p = t.plans[1];  // MIDDLE: slab product over q = k is Z[j, k, :]
  }
  // the tree contraction's workspace (its split-K partials, then its Ozaki
  // region) sits past every plain plan's: a deferred partial set of one
  // contraction never shares bytes with the Lo-slice region a solve writes
  // for another (SplitDefer::avoid would otherwise keep it undeferred)
  e->tree_base = align_up(e->ws_bytes, 256);
  e->ws_bytes = e->tree_base + tree_ws_offset(p, e->ld) + ozaki_ws_bytes(p, e->ld) + 256;
  CALS_CUDA_TRY(cudaMalloc(&e->d_partial, bytes));
  poison_alloc(e->d_partial, bytes);
  e->tree_variant = choose_variant(p.M, e->capacity, p.S);
  e->tree = choice;
  return kOk;
}

static int engine_free(Engine* e) {
  if (!e) return kOk;
  int prev = -1;
  cudaGetDevice(&prev);
  if (prev != e->device) cudaSetDevice(e->device);
  if (e->exec) cudaGraphExecDestroy(e->exec);
  if (e->graph) cudaGraphDestroy(e->graph);
  if (e->d_block) cudaFree(e->d_block);
  if (e->d_ws) cudaFree(e->d_ws);
  if (e->d_partial) cudaFree(e->d_partial);
  if (e->d_ones) cudaFree(e->d_ones);
  if (e->d_ls) cudaFree(e->d_ls);
  if (e->d_nnls) cudaFree(e->d_nnls);
  if (e->d_st) cudaFree(e->d_st);
  if (e->h_done) cudaFreeHost(e->h_done);
  if (e->h_st_pinned) cudaFreeHost(e->h_st_pinned);
  if (e->st_upload_ev) cudaEventDestroy(e->st_upload_ev);
  if (e->h_results) cudaFreeHost(e->h_results);
  for (int n = 0; n < kMaxOrder; ++n) {
    if (e->ev_fork[n]) cudaEventDestroy(e->ev_fork[n]);
    if (e->ev_join[n]) cudaEventDestroy(e->ev_join[n]);
  }
  if (e->side) cudaStreamDestroy(e->side);
  if (prev >= 0 && prev != e->device) cudaSetDevice(prev);
  delete e;
  return kOk;
}

static int engine_create(Tensor* t, int capacity, int n_models, const int* ranks, int trace_cap,
                         Engine** out) {
  CALS_CHECK(t && out && ranks, kErrInvalid, "null argument");
  CALS_CHECK(capacity >= 1, kErrInvalid, "capacity (r_star) must be >= 1");
  CALS_CHECK(n_models >= 0, kErrInvalid, "n_models must be >= 0");
  std::unique_ptr<Engine> e(new Engine());
  e->t = t;
  e->device = t->device;
  e->tensor_uid = t->uid;
  e->order = t->order;
  e->n_models = n_models;
  e->capacity = capacity;
  e->ranks.assign(ranks, ranks + n_models);
  const int N = t->order;
  int rmax = 1;
  long long rsum = 0;
  for (int k = 0; k < n_models; ++k) {
    CALS_CHECK(ranks[k] >= 1, kErrInvalid, "ranks must be >= 1");
    CALS_CHECK(ranks[k] <= capacity, kErrCapacity,
               "model rank " + std::to_string(ranks[k]) + " exceeds r_star " +
                   std::to_string(capacity));
    rmax = std::max(rmax, ranks[k]);
    rsum += ranks[k];
  }
  CALS_CHECK(rmax <= kMaxRank, kErrUnsupported,
             "ranks above " + std::to_string(kMaxRank) + " are not supported by the update kernel");
  e->max_rank = rmax;
  e->max_slots = std::max(1, std::min<int>(n_models, capacity));
  e->ld = align_up(capacity, 8);
  CALS_CHECK(e->ld * 8 <= 200 * 1024, kErrUnsupported, "r_star above 25600 is not supported");
  e->pool_off.resize((size_t)n_models * N);
  e->gram_off.resize(n_models);
  e->lam_off.resize(n_models);
  long long po = 0, go = 0, lo = 0;
  for (int k = 0; k < n_models; ++k) {
    for (int n = 0; n < N; ++n) {
      e->pool_off[(size_t)k * N + n] = po;
      po += t->dims[n] * ranks[k];
    }
    e->gram_off[k] = go;
    go += (long long)ranks[k] * ranks[k];
    e->lam_off[k] = lo;
    lo += ranks[k];
  }
  e->pool_elems = po;
  e->gram_stride = std::max<long long>(go, 1);
  CALS_CHECK(e->gram_stride < (1LL << 31), kErrUnsupported, "Gramian arena beyond 2^31 entries");
  e->lam_elems = std::max<long long>(lo, 1);
  e->trace_cap = std::max(trace_cap, 1);

  // launch geometry
  const int sms = sm_count(t->device);
  e->upd_grid = std::max(1, std::min(e->max_slots, sms * 4));
  e->upd_nthr = pick_nthr(rmax);
  e->upd_kernel = update_kernel_for(rmax, &e->upd_rb);
  e->upd_smem = (rmax > kSmemRankMax ? 0 : size_t(rmax) * rmax * 8) +
                std::max(size_t(rmax) * e->upd_nthr, size_t(kUpdThreads) * (e->upd_rb + 1)) * 8;
  e->move_smem = size_t(e->ld) * 8;
  long long rows_total = 0, maxI = 1;
  for (int n = 0; n < N; ++n) {
    rows_total += t->dims[n];
    maxI = std::max(maxI, t->dims[n]);
  }
  e->move_grid = (int)std::max<long long>(1, std::min<long long>(rows_total, sms * 8));
  CALS_CUDA_TRY(raise_smem_limit((const void*)e->upd_kernel, e->upd_smem));
  CALS_CUDA_TRY(raise_smem_limit((const void*)engine_move_kernel, e->move_smem));

  // arena layout
  struct Item { void** dst; size_t bytes; };
  EngState& h = e->h_st;
  std::memset(&h, 0, sizeof(h));
  long long fbytes_total = 0;
  std::vector<Item> items;
  const int ms = e->max_slots;
  const int mv = 2 * ms + 2;
  items.push_back({(void**)&h.slot_model, size_t(ms) * 4});
  items.push_back({(void**)&h.slot_off, size_t(ms) * 4});
  items.push_back({(void**)&h.slot_info, size_t(ms) * 16});
  items.push_back({(void**)&h.changed, 4});
  items.push_back({(void**)&h.lo_stale, 4});
  items.push_back({(void**)&h.mv_kind, size_t(mv) * 4});
  items.push_back({(void**)&h.mv_model, size_t(mv) * 4});
  items.push_back({(void**)&h.mv_src, size_t(mv) * 4});
  items.push_back({(void**)&h.mv_dst, size_t(mv) * 4});
  items.push_back({(void**)&h.mv_len, size_t(mv) * 4});
  items.push_back({(void**)&h.mv_pre, size_t(mv) * 4});
  const size_t nmod = std::max(1, n_models);
  items.push_back({(void**)&h.rank, nmod * 4});
  items.push_back({(void**)&h.pool_off, nmod * N * 8});
  items.push_back({(void**)&h.gram_off, nmod * 8});
  items.push_back({(void**)&h.status, nmod * 4});
  items.push_back({(void**)&h.iters, nmod * 4});
  items.push_back({(void**)&h.failed, nmod * 4});
  items.push_back({(void**)&h.fresh, nmod * 4});
  items.push_back({(void**)&h.retire_seq, nmod * 4});
  items.push_back({(void**)&h.f_prev, nmod * 8});
  items.push_back({(void**)&h.err, nmod * 8});
  items.push_back({(void**)&h.fit, nmod * 8});
  items.push_back({(void**)&h.t_admit, nmod * 8});
  items.push_back({(void**)&h.t_retire, nmod * 8});
  items.push_back({(void**)&h.grams, size_t(N) * e->gram_stride * 8});
  items.push_back({(void**)&h.pool, size_t(std::max<long long>(po, 1)) * 8});
  for (int n = 0; n < N; ++n) {
    items.push_back({(void**)&h.F[n], size_t(t->dims[n]) * e->ld * 8});
    fbytes_total += t->dims[n] * e->ld * 8;
  }
  items.push_back({(void**)&h.Mout, size_t(maxI) * e->ld * 8});
  items.push_back({(void**)&h.scratch, size_t(e->upd_grid) * upd_scratch_doubles(rmax) * 8});
  items.push_back({(void**)&h.tr_width, size_t(e->trace_cap) * 4});
  items.push_back({(void**)&h.tr_active, size_t(e->trace_cap) * 4});
  items.push_back({(void**)&h.tr_time, size_t(e->trace_cap) * 8});
  items.push_back({(void**)&e->d_lam, size_t(e->lam_elems) * 8});
  items.push_back({(void**)&e->d_lam_off, nmod * 8});
  // split update buffers
  // CALS_SPLIT_UPDATE=0 keeps the one-kernel (block per model) update
  const char* split_env = getenv("CALS_SPLIT_UPDATE");
  e->split = rmax <= kFastR && (!split_env || atoi(split_env) != 0);
  int nch_max = 1;
  for (int n = 0; n < N; ++n) {
    e->nch[n] = int((t->dims[n] + kSolveRows - 1) / kSolveRows);
    nch_max = std::max(nch_max, e->nch[n]);
  }
  UpdArgs& ua = e->ua;
  items.push_back({(void**)&ua.pflag, nmod * 4});
  items.push_back({(void**)&h.arrive, nmod * 4});
  items.push_back({(void**)&h.solbad, nmod * 4});
  items.push_back({(void**)&ua.ubuf, 3 * size_t(e->gram_stride) * 8});
  items.push_back({(void**)&ua.gpart, size_t(e->gram_stride) * nch_max * 8});
  items.push_back({(void**)&ua.ipart, nmod * nch_max * 8});
  size_t total = 0;
  for (auto& it : items) total = align_up(total, 256) + it.bytes;
  CALS_CUDA_TRY(cudaMalloc(&e->d_block, total));
  poison_alloc(e->d_block, total);
  CALS_CUDA_TRY(cudaMemset(e->d_block, 0, total));
  size_t off = 0;
  for (auto& it : items) {
    off = align_up(off, 256);
    *it.dst = static_cast<char*>(e->d_block) + off;
    off += it.bytes;
  }
  CALS_CUDA_TRY(cudaMalloc(&e->d_st, sizeof(EngState)));
  poison_alloc(e->d_st, sizeof(EngState));
  // split update: kernel-parameter block (constant bank) of device pointers
  ua.st = e->d_st;
  ua.n_active = &e->d_st->n_active;
  ua.rev = [] {
    const char* v = getenv("CALS_SOLVE_REV");
    return !v || atoi(v) != 0;
  }() ? 1 : 0;
  ua.slot_info = h.slot_info;
  ua.failed = h.failed;
  ua.fresh = h.fresh;
  ua.arrive = h.arrive;
  ua.solbad = h.solbad;
  ua.grams = h.grams;
  ua.gram_stride = e->gram_stride;
  ua.Mout = h.Mout;
  for (int n = 0; n < N; ++n) {
    ua.F[n] = h.F[n];
    ua.dims[n] = t->dims[n];
  }
  ua.ld = e->ld;
  ua.order = N;
  ua.lo[0].src = -1;
  ua.lo[1].src = -1;
  ua.lo_stale = h.lo_stale;
  if (e->split) {
    split_kernels_for(e->upd_rb, &e->prep_kernel, &e->solve_kernel, &e->solve_last_kernel,
                      &e->solve_smem);
    CALS_CUDA_TRY(raise_smem_limit((const void*)e->solve_kernel, e->solve_smem));
    CALS_CUDA_TRY(raise_smem_limit((const void*)e->solve_last_kernel, e->solve_smem));
    CALS_CUDA_TRY(cudaStreamCreateWithFlags(&e->side, cudaStreamNonBlocking));
    for (int n = 0; n < N; ++n) {
      CALS_CUDA_TRY(cudaEventCreateWithFlags(&e->ev_fork[n], cudaEventDisableTiming));
      CALS_CUDA_TRY(cudaEventCreateWithFlags(&e->ev_join[n], cudaEventDisableTiming));
    }
  }
  CALS_CUDA_TRY(cudaHostAlloc(&e->h_done, 64, cudaHostAllocMapped));
  CALS_CUDA_TRY(cudaHostAlloc(&e->h_st_pinned, sizeof(EngState), cudaHostAllocDefault));
  CALS_CUDA_TRY(cudaEventCreateWithFlags(&e->st_upload_ev, cudaEventDisableTiming));
  CALS_CUDA_TRY(cudaHostGetDevicePointer(&e->d_done_alias, e->h_done, 0));

  // constant tables
  if (n_models > 0) {
    CALS_CUDA_TRY(cudaMemcpy((void*)h.rank, ranks, size_t(n_models) * 4, cudaMemcpyHostToDevice));
    CALS_CUDA_TRY(cudaMemcpy((void*)h.pool_off, e->pool_off.data(), size_t(n_models) * N * 8,
                             cudaMemcpyHostToDevice));
    CALS_CUDA_TRY(cudaMemcpy((void*)h.gram_off, e->gram_off.data(), size_t(n_models) * 8,
                             cudaMemcpyHostToDevice));
    CALS_CUDA_TRY(cudaMemcpy(e->d_lam_off, e->lam_off.data(), size_t(n_models) * 8,
                             cudaMemcpyHostToDevice));
  }
  h.order = N;
  h.n_models = n_models;
  h.capacity = capacity;
  h.max_slots = ms;
  h.max_rank = rmax;
  h.ld = e->ld;
  for (int n = 0; n < N; ++n) h.dims[n] = t->dims[n];
  h.gram_stride = e->gram_stride;
  h.tr_cap = e->trace_cap;
  h.host_done = e->d_done_alias;

  // MTTKRP workspace + variants (chosen for the capacity width)
  e->ws_bytes = 256;
  for (int n = 0; n < N; ++n) {
    e->ws_bytes = std::max(e->ws_bytes, mttkrp_workspace_bytes(*t, n, e->ld));
    e->variants[n] = choose_variant(t->plans[n].M, capacity, t->plans[n].S);
  }
  int rc = setup_tree(e.get());
  if (rc) return rc;
  CALS_CUDA_TRY(cudaMalloc(&e->d_ws, e->ws_bytes));
  poison_alloc(e->d_ws, e->ws_bytes);
  *out = e.release();
  return kOk;
}

// Per-model run state to its initial values (driver.py:56-67): status,
// iteration count, failure / fresh flags 0, retirement order -1, f_prev =
// -inf, error = +inf, fit = -inf.
__global__ void engine_reset_kernel(const EngState h, int nm) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *h.changed = 0;
    *h.lo_stale = 1;
  }
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nm; k += gridDim.x * blockDim.x) {
    h.status[k] = 0;
    h.iters[k] = 0;
    h.failed[k] = 0;
    h.fresh[k] = 0;
    h.arrive[k] = 0;
    h.solbad[k] = 0;
    if (h.has_snap) h.has_snap[k] = 0;
    h.retire_seq[k] = -1;
    h.f_prev[k] = -INFINITY;
    h.err[k] = INFINITY;
    h.fit[k] = -INFINITY;
  }
}

// Stream-ordered, no host synchronisation: the state goes up from a
// page-locked copy (the previous upload from it has completed -- every run
// ends with a stream sync, and the event guards the step-wise API), the
// per-model arrays are reset by one kernel.
static int engine_reset(Engine* e, double tol, int max_iterations, double sqnorm,
                        cudaStream_t stream) {
  EngState& h = e->h_st;
  h.width = h.n_active = h.queue_head = h.n_retired = h.plans_done = h.done = 0;
  h.old_width = h.n_moves = h.move_elems = 0;
  h.tol = tol;
  h.max_iterations = max_iterations;
  h.sqnorm = sqnorm;
  const int nm = std::max(1, e->n_models);
  CALS_CUDA_TRY(cudaEventSynchronize(e->st_upload_ev));
  *e->h_st_pinned = h;
  CALS_CUDA_TRY(cudaMemcpyAsync(e->d_st, e->h_st_pinned, sizeof(EngState), cudaMemcpyHostToDevice,
                                stream));
  CALS_CUDA_TRY(cudaEventRecord(e->st_upload_ev, stream));
  engine_reset_kernel<<<std::max(1, std::min((nm + 255) / 256, 148)), 256, 0, stream>>>(h, nm);
  CALS_CUDA_TRY(cudaGetLastError());
  e->h_done[1] = 0;
  *(volatile int*)e->h_done = 0;
  return kOk;
}

// Driver iterations a run takes when no model can stop early (tol <= 0: every
// admitted model runs exactly max_iterations): the FIFO admission with
// head-of-line blocking (plan kernel) replayed on the host.  Failures can only
// shorten the run (the extra iterations are no-ops on the device).
static long long fixed_iteration_count(const Engine* e, int max_iterations) {
  std::vector<std::pair<int, int>> active;  // (rank, iterations left)
  int head = 0;
  long long width = 0, graphs = 0;
  auto admit = [&] {
    while (head < e->n_models && width + e->ranks[head] <= e->capacity) {
      active.push_back({e->ranks[head], max_iterations});
      width += e->ranks[head++];
    }
  };
  admit();
  while (!active.empty()) {
    ++graphs;
    std::vector<std::pair<int, int>> keep;
    for (auto& a : active) {
      if (--a.second > 0)
        keep.push_back(a);
      else
        width -= a.first;
    }
    active.swap(keep);
    admit();
    if (active.empty() && head < e->n_models) return 0;  // blocked: let the device decide
  }
  return graphs;
}

// M_n -> Mout for the current layout (dimension-tree aware).  With `defer`, a
// split-K contraction leaves M_n as partials for the solve kernel instead.
static int enqueue_mode_mttkrp(Engine* e, int n, cudaStream_t stream,
                               SplitDefer* defer = nullptr) {
  Tensor& t = *e->t;
  const int N = e->order;
  FactorSet fs{};
  for (int i = 0; i < N; ++i) fs.ptr[i] = e->h_st.F[i];
  fs.ld = e->ld;
  const int* wptr = &e->d_st->width;
  const int sms = sm_count(t.device);
  double* const* F = e->h_st.F;
  double* Mo = e->h_st.Mout;
  const long long ld = e->ld, cap = e->capacity;
  void* oz_ws = nullptr;
  size_t oz_bytes = 0;
  if (e->tree != kTreeNone) {
    oz_bytes = ozaki_ws_bytes(e->tree_plan, ld);
    oz_ws = tree_ws(e) + tree_ws_offset(e->tree_plan, ld);
  }
  {
    int rc = kOk;
    if (e->tree == kTreeY && n == 0) {
      // M0 = sum_j A1[j] (sum_k X[:,j,k] A2[k]); the inner slab products are
      // the partial Y[i + I0p j] kept for mode 1
      rc = launch_contraction(t, e->tree_plan, 100, F[2], t.dims[2], ld, F[1], ld, 0, wptr, cap,
                              Mo, ld, reinterpret_cast<double*>(tree_ws(e)), e->tree_variant, stream, e->d_partial, ld, t.i0p,
                              oz_ws, oz_bytes, false, e->lo_carry ? e->h_st.lo_stale : nullptr,
                              defer);
    } else if (e->tree == kTreeY && n == 1) {
      // M1 = Y x_i A0(new): A2 unchanged since Y was formed
      rc = launch_partial_ttv(e->d_partial, ld, t.i0p, t.dims[1], 0, t.dims[0], F[0], ld, 0,
                              wptr, cap, t.dims[1], Mo, ld, sms, stream);
    } else if (e->tree == kTreeZ && n == 1) {
      // M1 = sum_k A2[k] (sum_i X[i,:,k] A0(new)[i]); slab products = Z[j + I1 k]
      rc = launch_contraction(t, e->tree_plan, 1, F[0], t.dims[0], ld, F[2], ld, 0, wptr, cap, Mo,
                              ld, reinterpret_cast<double*>(tree_ws(e)), e->tree_variant, stream, e->d_partial, ld, t.dims[1],
                              oz_ws, oz_bytes, n == e->lo_target, nullptr, defer);
    } else if (e->tree == kTreeZ && n == 2) {
      // M2 = Z x_j A1(new): A0 unchanged since Z was formed
      rc = launch_partial_ttv(e->d_partial, ld, t.dims[1], t.dims[2], 0, t.dims[1], F[1], ld, 0,
                              wptr, cap, t.dims[2], Mo, ld, sms, stream);
    } else {
      rc = launch_mttkrp(t, n, fs, 0, wptr, cap, Mo, ld, e->d_ws, e->ws_bytes, e->variants[n],
                         stream, n == e->lo_target,
                         (n == 0 && e->lo_carry) ? e->h_st.lo_stale : nullptr, defer);
    }
    if (rc) return rc;
  }
  return kOk;
}

static int enqueue_mode_update(Engine* e, int n, cudaStream_t stream) {
  e->upd_kernel<<<e->upd_grid, kUpdThreads, e->upd_smem, stream>>>(e->d_st, e->h_st.slot_info,
                                                                   n, e->upd_nthr);
  CALS_CUDA_TRY(cudaGetLastError());
  return kOk;
}

static int enqueue_plan(Engine* e, cudaStream_t stream) {
  CALS_CUDA_TRY(launch_dep(engine_plan_kernel, dim3(1), dim3(kPlanThreads), 0, stream, e->d_st));
  CALS_CUDA_TRY(launch_dep(engine_move_kernel, dim3(e->move_grid), dim3(256), e->move_smem, stream,
                           e->d_st));
  return kOk;
}

// Line search: candidates + their Gramians, ONE fused last-mode MTTKRP over
// every candidate at once (the reference runs one single-instance MTTKRP per
// model, driver.py:252-254), then accept / stopping rule / snapshot.
static int enqueue_line_search(Engine* e, cudaStream_t stream) {
  const int N = e->order;
  ls_candidate_kernel<<<e->upd_grid, kUpdThreads, e->ls_smem, stream>>>(e->d_st);
  CALS_CUDA_TRY(cudaGetLastError());
  FactorSet fs{};
  for (int n = 0; n < N; ++n) fs.ptr[n] = e->h_st.Cb[n];
  fs.ld = e->ld;
  int rc = launch_mttkrp(*e->t, N - 1, fs, 0, &e->d_st->width, e->capacity, e->h_st.Mout, e->ld,
                         e->d_ws, e->ws_bytes, e->variants[N - 1], stream);
  if (rc) return rc;
  ls_finish_kernel<<<e->upd_grid, kUpdThreads, 0, stream>>>(e->d_st);
  CALS_CUDA_TRY(cudaGetLastError());
  return kOk;
}

// CALS_PDL=0 disables programmatic dependent launches (A/B measurements)
bool pdl_enabled() {
  static const bool on = [] {
    const char* v = getenv("CALS_PDL");
    return !v || atoi(v) != 0;
  }();
  return on;
}

// CALS_DEFER_REDUCE=0 keeps split_reduce_kernel in front of every solve (A/B)
static bool defer_reduce_enabled() {
  static const bool on = [] {
    const char* v = getenv("CALS_DEFER_REDUCE");
    return !v || atoi(v) != 0;
  }();
  return on;
}

// Split update of mode n: prep(n) forked onto the side stream before the
// MTTKRP of mode n is queued (it depends only on what the main stream has
// done so far), solve(n) after both.
static int enqueue_split_mode(Engine* e, int n, cudaStream_t stream) {
  CALS_CUDA_TRY(cudaEventRecord(e->ev_fork[n], stream));
  CALS_CUDA_TRY(cudaStreamWaitEvent(e->side, e->ev_fork[n], 0));
  e->prep_kernel<<<e->max_slots, kPrepThreads, 0, e->side>>>(e->ua, n);
  CALS_CUDA_TRY(cudaGetLastError());
  CALS_CUDA_TRY(cudaEventRecord(e->ev_join[n], e->side));
  // non-last modes: the solve sums the split-K partials itself (the last
  // mode's M also feeds the fit's <A, M>, read after the solve)
  SplitDefer defer;
  const bool defer_ok = n < e->order - 1 && defer_reduce_enabled() &&
                        (long long)e->t->dims[n] * e->ld < (1LL << 31);
  // the solve of mode n writes its fused Lo-slice targets while other CTAs
  // of the same launch still stage M_n from the partials: never defer into
  // a partial set that shares bytes with a target
  for (int t = 0; t < 2; ++t) {
    const UpdArgs::LoTarget& tg = e->ua.lo[t];
    if (tg.src != n) continue;
    defer.add_avoid(tg.ls, size_t(7) * size_t(tg.stride));  // 7 Ozaki slices (oz::kSlices)
    defer.add_avoid(tg.cex, size_t(e->capacity + 256) * sizeof(int));
    defer.add_avoid(tg.queue, sizeof(int));
  }
  int rc = enqueue_mode_mttkrp(e, n, stream, defer_ok ? &defer : nullptr);
  if (rc) return rc;
  UpdArgs ua = e->ua;
  ua.mpart = defer.part;
  ua.mpart_stride = defer.stride;
  ua.mpart_ld = defer.ldp;
  ua.mS = defer.S;
  CALS_CUDA_TRY(cudaStreamWaitEvent(stream, e->ev_join[n], 0));
  SolveKernel k = n == e->order - 1 ? e->solve_last_kernel : e->solve_kernel;
  // programmatic launch: the solve's prologue (slot, pflag, U) overlaps the
  // tail of the kernel that produces M_n (griddep_wait before reading it)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(e->max_slots * e->nch[n]);
  cfg.blockDim = dim3(kSolveRows);
  cfg.dynamicSmemBytes = e->solve_smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CALS_CUDA_TRY(cudaLaunchKernelEx(&cfg, k, ua, n, e->nch[n]));
#ifdef CALS_SOLVE_PROFILE
  // profiling aid: a non-last solve is idempotent (reads M and U, rewrites
  // the same rows, Gramian and slices), so a second launch right behind the
  // first shows the phase stamps with a warm instruction cache
  if (getenv("CALS_SOLVE_TWICE") && n < e->order - 1)
    CALS_CUDA_TRY(cudaLaunchKernelEx(&cfg, k, ua, n, e->nch[n]));
#endif
  return kOk;
}

static int enqueue_iteration(Engine* e, cudaStream_t stream) {
  const bool split = e->split && !e->h_st.nonneg;
  for (int n = 0; n < e->order; ++n) {
    int rc = split ? enqueue_split_mode(e, n, stream) : enqueue_mode_mttkrp(e, n, stream);
    if (!rc && !split) rc = enqueue_mode_update(e, n, stream);
    if (rc) return rc;
  }
  if (e->h_st.ls_enabled) {
    int rc = enqueue_line_search(e, stream);
    if (rc) return rc;
  }
  return enqueue_plan(e, stream);
}

static int engine_set_nonneg(Engine* e, int enabled) {
  EngState& h = e->h_st;
  if (enabled) {
    CALS_CHECK(e->max_rank <= kFastR, kErrUnsupported,
               "non-negative updates support ranks up to 32");
    if (!e->d_nnls) {
      const int N = e->order;
      const size_t nm = std::max(1, e->n_models);
      std::vector<long long> offs(nm * N, 0);
      long long at = 0;
      for (int k = 0; k < e->n_models; ++k)
        for (int n = 0; n < N; ++n) {
          offs[(size_t)k * N + n] = at;
          at += e->t->dims[n];
        }
      const size_t b_state = align_up(size_t(std::max<long long>(at, 1)) * 4, 256);
      const size_t b_off = align_up(offs.size() * 8, 256);
      CALS_CUDA_TRY(cudaMalloc(&e->d_nnls, b_state + b_off + nm * 4));
      poison_alloc(e->d_nnls, b_state + b_off + nm * 4);
      CALS_CUDA_TRY(cudaMemset(e->d_nnls, 0, b_state + b_off + nm * 4));
      h.nnls_state = static_cast<unsigned*>(e->d_nnls);
      h.nnls_off = reinterpret_cast<long long*>(static_cast<char*>(e->d_nnls) + b_state);
      h.nnls_warn = reinterpret_cast<int*>(static_cast<char*>(e->d_nnls) + b_state + b_off);
      CALS_CUDA_TRY(cudaMemcpy((void*)h.nnls_off, offs.data(), offs.size() * 8,
                               cudaMemcpyHostToDevice));
    }
    const size_t need = size_t(e->max_rank) * e->max_rank * 8 +
                        size_t(kUpdThreads / 32) * kNnlsWs * 8;
    if (need > e->upd_smem) {
      e->upd_smem = need;
      CALS_CUDA_TRY(raise_smem_limit((const void*)e->upd_kernel, e->upd_smem));
    }
  }
  if (h.nonneg != (enabled ? 1 : 0)) {
    if (e->exec) cudaGraphExecDestroy(e->exec);
    if (e->graph) cudaGraphDestroy(e->graph);
    e->exec = nullptr;
    e->graph = nullptr;
  }
  h.nonneg = enabled ? 1 : 0;
  return kOk;
}

static int engine_set_line_search(Engine* e, int enabled, double alpha) {
  EngState& h = e->h_st;
  if (enabled && !e->d_ls) {
    const int N = e->order;
    const size_t nm = std::max(1, e->n_models);
    size_t total = 0;
    std::vector<std::pair<void**, size_t>> items;
    for (int n = 0; n < N; ++n) {
      items.push_back({(void**)&h.S[n], size_t(e->t->dims[n]) * e->ld * 8});
      items.push_back({(void**)&h.Cb[n], size_t(e->t->dims[n]) * e->ld * 8});
    }
    items.push_back({(void**)&h.cgrams, size_t(N) * e->gram_stride * 8});
    items.push_back({(void**)&h.has_snap, nm * 4});
    items.push_back({(void**)&h.ls_act, nm * 4});
    items.push_back({(void**)&h.e_tmp, nm * 8});
    for (auto& it : items) total = align_up(total, 256) + it.second;
    CALS_CUDA_TRY(cudaMalloc(&e->d_ls, total));
    poison_alloc(e->d_ls, total);
    CALS_CUDA_TRY(cudaMemset(e->d_ls, 0, total));
    size_t off = 0;
    for (auto& it : items) {
      off = align_up(off, 256);
      *it.first = static_cast<char*>(e->d_ls) + off;
      off += it.second;
    }
    e->ls_smem = size_t(kUpdThreads) * (kFastR + 1) * 8;
    CALS_CUDA_TRY(raise_smem_limit((const void*)ls_candidate_kernel, e->ls_smem));
  }
  if (h.ls_enabled != enabled || (enabled && h.ls_alpha != alpha)) {
    // the captured iteration graph depends on the line-search setting
    if (e->exec) cudaGraphExecDestroy(e->exec);
    if (e->graph) cudaGraphDestroy(e->graph);
    e->exec = nullptr;
    e->graph = nullptr;
  }
  h.ls_enabled = enabled ? 1 : 0;
  h.ls_alpha = alpha;
  return kOk;
}

static int engine_capture(Engine* e, cudaStream_t stream) {
  if (e->exec && !e->graph_stale) return kOk;
  // capture on a private stream (the caller's stream may be the legacy default stream)
  cudaStream_t cs;
  CALS_CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  CALS_CUDA_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
  int rc = enqueue_iteration(e, cs);
  cudaGraph_t g = nullptr;
  cudaError_t ce = cudaStreamEndCapture(cs, &g);
  cudaStreamDestroy(cs);
  if (rc) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  CALS_CUDA_TRY(ce);
  if (e->exec) {
    // stale graph (new tensor): update the instantiated graph in place
    cudaGraphExecUpdateResultInfo info;
    if (cudaGraphExecUpdate(e->exec, g, &info) == cudaSuccess) {
      if (e->graph) cudaGraphDestroy(e->graph);
      e->graph = g;
      e->graph_stale = false;
      return kOk;
    }
    (void)cudaGetLastError();
    cudaGraphExecDestroy(e->exec);
    e->exec = nullptr;
    if (e->graph) cudaGraphDestroy(e->graph);
    e->graph = nullptr;
  }
  e->graph = g;
  CALS_CUDA_TRY(cudaGraphInstantiate(&e->exec, g, 0));
  e->graph_stale = false;
  (void)stream;
  return kOk;
}

// Kernel nodes of the captured iteration graph (prep on the side stream
// included): what one cudaGraphLaunch puts on the GPU.
static int count_graph_kernels(cudaGraph_t g) {
  size_t n = 0;
  if (!g || cudaGraphGetNodes(g, nullptr, &n) != cudaSuccess) return 0;
  std::vector<cudaGraphNode_t> nodes(n);
  if (cudaGraphGetNodes(g, nodes.data(), &n) != cudaSuccess) return 0;
  int k = 0;
  for (auto nd : nodes) {
    cudaGraphNodeType ty;
    if (cudaGraphNodeGetType(nd, &ty) == cudaSuccess && ty == cudaGraphNodeTypeKernel) ++k;
  }
  return k;
}

// Run every queued model to retirement.  `pool` must already hold the
// starting factors (per model, per mode, row-major I_n x R_k).
// Lo-slice fusion (UpdArgs::lo): when the first contraction after mode 0
// takes F[0] (just solved) as its Lo operand and runs on the INT8 path, the
// mode-0 solve kernel writes that contraction's Lo slices, exponents and
// unit counter, and the contraction skips its slicing kernel (one launch and
// one pass over the factor less per iteration; identical slices).  Only on the
// plain split-update path (no line search / NNLS, whose extra contractions
// share the workspace) with single-chunk mode-0 solves.  CALS_FUSE_LO=0
// disables it.
static void setup_lo_fusion(Engine* e) {
  e->lo_target = -1;
  e->lo_carry = false;
  e->ua.lo[0].src = -1;
  e->ua.lo[1].src = -1;
  e->ua.lo_stale = e->h_st.lo_stale;
  const char* env = getenv("CALS_FUSE_LO");
  if (env && atoi(env) == 0) return;
  if (!e->split || e->h_st.nonneg || e->h_st.ls_enabled || e->order != 3) return;
  Tensor& t = *e->t;
  auto fill = [&](UpdArgs::LoTarget& tg, const ModePlan& p, int lo_mode, void* ws, int src) {
    const OzLoLayout l = ozaki_lo_layout(p, t.dims[lo_mode], e->capacity, ws);
    tg.ls = l.ls;
    tg.cex = l.cex;
    tg.queue = l.queue;
    tg.stride = l.slice_stride;
    tg.Kp = l.Kp;
    tg.Dp = l.Dp;
    tg.src = src;
  };
  // target 0: the first contraction after mode 0 that takes F[0] as Lo
  if (e->nch[0] == 1) {
    for (int n = 1; n < e->order; ++n) {
      if ((e->tree == kTreeY && n == 1) || (e->tree == kTreeZ && n == 2)) continue;  // TTV
      const ModePlan* p;
      void* ws;
      if (e->tree == kTreeZ && n == 1) {  // Z = X x_1 A0(new): Lo = F[0]
        p = &e->tree_plan;
        ws = tree_ws(e) + tree_ws_offset(e->tree_plan, e->ld);
      } else {
        p = &t.plans[n];
        if (!p->lo_direct() || p->lo_modes[0] != 0) break;
        ws = mttkrp_oz_ws(t, n, e->ld, e->d_ws, e->ws_bytes);
      }
      if (ws && ozaki_ready(t, *p, n)) {
        fill(e->ua.lo[0], *p, 0, ws, 0);
        e->lo_target = n;
      }
      break;
    }
  }
  // target 1 (carry): the next iteration's mode-0 contraction, written by the
  // solve of its Lo mode when nothing between that solve and mode 0 contracts
  // through the shared workspace (tree schedules: the modes in between are a
  // TTV); its slicing kernel still runs whenever the plan moved columns
  {
    const ModePlan* p = nullptr;
    void* ws = nullptr;
    int key = 0, src = -1;
    if (e->tree == kTreeY) {  // mode 0: Y-tree contraction, Lo = F[2]
      p = &e->tree_plan;
      key = 100;
      src = 2;
      ws = tree_ws(e) + tree_ws_offset(e->tree_plan, e->ld);
    } else if (e->tree == kTreeZ && t.plans[0].lo_direct()) {  // mode 0 plain, mode 2 a TTV
      p = &t.plans[0];
      key = 0;
      src = t.plans[0].lo_modes[0];
      ws = mttkrp_oz_ws(t, 0, e->ld, e->d_ws, e->ws_bytes);
    }
    if (p && src > 0 && src < e->order && e->nch[src] == 1 && ws && ozaki_ready(t, *p, key)) {
      fill(e->ua.lo[1], *p, src, ws, src);
      e->ua.lo[1].queue = nullptr;  // zeroed by the (always launched) slicing kernel
      e->lo_carry = true;
    }
  }
}

static int engine_run(Engine* e, double tol, int max_iterations, double sqnorm, int use_graph,
                      cudaStream_t stream, int* iterations_out) {
  CALS_CHECK(max_iterations >= 1, kErrInvalid, "max_iterations must be >= 1");
  CALS_CHECK(sqnorm > 0.0, kErrInvalid, "tensor squared norm must be positive");
  int rc = engine_reset(e, tol, max_iterations, sqnorm, stream);
  if (rc) return rc;
  if (e->n_models == 0) {
    if (iterations_out) *iterations_out = 0;
    return kOk;
  }
  rc = engine_prepare_slices(e, stream);
  if (rc) return rc;
  setup_lo_fusion(e);
  // initial admission
  CALS_CUDA_TRY(launch_dep(engine_plan_kernel, dim3(1), dim3(kPlanThreads), 0, stream, e->d_st));
  CALS_CUDA_TRY(launch_dep(engine_move_kernel, dim3(e->move_grid), dim3(256), e->move_smem, stream,
                           e->d_st));
  CALS_CUDA_TRY(cudaGetLastError());
  if (use_graph) {
    rc = engine_capture(e, stream);
    if (rc) return rc;
    e->graph_kernels = count_graph_kernels(e->graph);
  }
  // tol <= 0: the iteration count is known, so the graphs go out back to back
  // (no completion polling, no trailing no-op iterations)
  const long long exact = (use_graph && tol <= 0.0) ? fixed_iteration_count(e, max_iterations) : 0;
  const int kLook = 3;
  cudaEvent_t ev[kLook];
  for (int i = 0; i < kLook; ++i)
    CALS_CUDA_TRY(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
  long long launched = 0;
  // Upper bound on driver iterations: every model needs <= max_iterations.
  const long long bound = (long long)max_iterations * std::max(1, e->n_models) + 2;
  int result = kOk;
  while (launched < bound) {
    if (use_graph) {
      cudaError_t ce = cudaGraphLaunch(e->exec, stream);
      if (ce != cudaSuccess) {
        set_error(std::string("cudaGraphLaunch: ") + cudaGetErrorString(ce));
        result = kErrCuda;
        break;
      }
    } else {
      rc = enqueue_iteration(e, stream);
      if (rc) { result = rc; break; }
    }
    cudaEventRecord(ev[launched % kLook], stream);
    ++launched;
    if (launched < exact) continue;
    if (launched == exact) {
      cudaError_t ce = cudaStreamSynchronize(stream);
      if (ce != cudaSuccess) {
        set_error(std::string("engine iteration failed: ") + cudaGetErrorString(ce));
        result = kErrCuda;
        break;
      }
      if (*(volatile int*)e->h_done) break;
      continue;  // not done (should not happen): poll as for tol > 0
    }
    if (launched >= kLook) {
      cudaError_t ce = cudaEventSynchronize(ev[(launched - kLook) % kLook]);
      if (ce != cudaSuccess) {
        set_error(std::string("engine iteration failed: ") + cudaGetErrorString(ce));
        result = kErrCuda;
        break;
      }
      if (*(volatile int*)e->h_done) break;
    }
  }
  cudaError_t ce = cudaStreamSynchronize(stream);
  for (int i = 0; i < kLook; ++i) cudaEventDestroy(ev[i]);
  if (result) return result;
  CALS_CUDA_TRY(ce);
  CALS_CHECK(*(volatile int*)e->h_done, kErrInvalid, "engine did not terminate");
  const int plans = ((volatile int*)e->h_done)[1];
  e->last_iterations = plans - 1;
  // reset + initial plan + move, then one graph per launched iteration
  e->last_launches = 3 + (use_graph ? launched * e->graph_kernels : 0);
  if (iterations_out) *iterations_out = plans - 1;
  return kOk;
}

}  // namespace cals

// ============================================================ C ABI ========
#include "../../include/cals_b200.h"

using namespace cals;

#ifdef CALS_SOLVE_PROFILE
namespace cals { int debug_solve_prof(long long* host, size_t bytes); }
#endif
struct cals_tensor { Tensor* t; };
struct cals_engine { Engine* e; };

extern "C" {

#ifdef CALS_SOLVE_PROFILE
int cals_debug_solve_prof(long long* host, size_t bytes) {
  return cals::debug_solve_prof(host, bytes);
}
#endif
#ifdef CALS_UPD_PROFILE
// profiling builds only (not in the public header): the update kernel's
// per-(mode, slot) phase stamps of the last launches
int cals_debug_upd_prof(long long* host, size_t bytes) {
  CALS_CUDA_TRY(cudaMemcpyFromSymbol(host, g_upd_prof, std::min(bytes, sizeof(g_upd_prof))));
  return kOk;
}
#endif

int cals_abi_version(void) { return CALS_B200_ABI_VERSION; }

const char* cals_last_error(void) { return get_error(); }

int cals_tensor_create(int order, const int64_t* dims, const double* host_data,
                       const double* device_data, void* stream, cals_tensor** out) {
  Tensor* t = nullptr;
  int rc = tensor_create(order, dims, host_data, device_data, (cudaStream_t)stream, &t);
  if (rc) return rc;
  *out = new cals_tensor{t};
  return kOk;
}

int cals_tensor_destroy(cals_tensor* t) {
  if (t) {
    tensor_destroy(t->t);
    delete t;
  }
  return kOk;
}

int cals_tensor_sqnorm(cals_tensor* t, void* stream, double* out) {
  CALS_CHECK(t && out, kErrInvalid, "null argument");
  return tensor_sqnorm(t->t, (cudaStream_t)stream, out);
}

int cals_tensor_data(cals_tensor* t, double** data, int64_t* padded_i0) {
  CALS_CHECK(t, kErrInvalid, "null tensor");
  if (data) *data = t->t->data;
  if (padded_i0) *padded_i0 = t->t->i0p;
  return kOk;
}

int cals_mttkrp_workspace_bytes(cals_tensor* t, int mode, int64_t capacity, size_t* bytes) {
  CALS_CHECK(t && bytes, kErrInvalid, "null argument");
  CALS_CHECK(mode >= 0 && mode < t->t->order, kErrInvalid, "mode out of range");
  *bytes = mttkrp_workspace_bytes(*t->t, mode, (capacity + 1) / 2 * 2);
  return kOk;
}

int cals_mttkrp(cals_tensor* t, int mode, int width, const double* const* factors, int64_t ldf,
                double* out, int64_t ldo, double* workspace, size_t workspace_bytes,
                int variant, void* stream) {
  CALS_CHECK(t && factors && out, kErrInvalid, "null argument");
  CALS_CHECK(mode >= 0 && mode < t->t->order, kErrInvalid, "mode out of range");
  CALS_CHECK(width >= 1 && width <= ldf, kErrInvalid, "width must be in [1, ldf]");
  CALS_CHECK(variant < num_variants(), kErrInvalid, "unknown variant");
  { const int rc_ = check_current_device(*t->t); if (rc_) return rc_; }
  FactorSet fs{};
  for (int n = 0; n < t->t->order; ++n) fs.ptr[n] = factors[n];
  fs.ld = ldf;
  return launch_mttkrp(*t->t, mode, fs, width, nullptr, ldf, out, ldo, workspace,
                       workspace_bytes, variant, (cudaStream_t)stream);
}

int cals_mttkrp_kernel_info(cals_tensor* t, int mode, int64_t width, int32_t* kernel,
                            double* tensor_ops) {
  CALS_CHECK(t && kernel && tensor_ops, kErrInvalid, "null argument");
  CALS_CHECK(mode >= 0 && mode < t->t->order, kErrInvalid, "mode out of range");
  CALS_CHECK(width >= 1, kErrInvalid, "width must be >= 1");
  const ModePlan& p = t->t->plans[mode];
  bool int8 = ozaki_eligible(p);
  if (int8) {
    // data-dependent part of the choice: the tensor slices are built (once)
    // and checked -- non-finite entries, scales beyond 2^+-900 and the
    // dynamic-range guard send the view to the FP64 kernel
    const int rc = ozaki_prepare(*t->t, p, mode, (cudaStream_t)0, true);
    if (rc) return rc;
    std::lock_guard<std::mutex> lk(t->t->mu);
    int8 = t->t->oz.count(mode) != 0;
  }
  if (int8) {
    *kernel = 1;
    *tensor_ops = ozaki_tensor_ops(p, width);
  } else {
    *kernel = 0;
    const VariantInfo& v = variant_info(choose_variant(p.M, width, p.S));
    const double mp = double((p.M + v.BM - 1) / v.BM * v.BM);
    const double wp = double((width + v.BN - 1) / v.BN * v.BN);
    *tensor_ops = 2.0 * mp * wp * double((p.Dp + 3) / 4 * 4) * double(p.Dq);
  }
  return kOk;
}

int cals_mttkrp_variants(int* count) {
  CALS_CHECK(count, kErrInvalid, "null argument");
  *count = num_variants();
  return kOk;
}

int cals_update_factor(int rows, int rank, const double* m, int64_t ldm, const double* h,
                       double* a, int64_t lda, double* scratch, int* status, void* stream) {
  CALS_CHECK(rows >= 0 && rank >= 1 && rank <= kMaxRank, kErrInvalid,
             "rank must be in [1, " + std::to_string(kMaxRank) + "]");
  CALS_CHECK(m && h && a && scratch && status, kErrInvalid, "null argument");
  const int nthr = pick_nthr(rank);
  const size_t smem =
      (rank > kSmemRankMax ? 0 : size_t(rank) * rank * 8) + size_t(rank) * nthr * 8;
  CALS_CUDA_TRY(raise_smem_limit((const void*)standalone_update_kernel, smem));
  standalone_update_kernel<<<1, kUpdThreads, smem, (cudaStream_t)stream>>>(
      m, ldm, rows, rank, h, a, lda, scratch, nthr, status);
  CALS_CUDA_TRY(cudaGetLastError());
  return kOk;
}

size_t cals_update_scratch_bytes(int rank) { return size_t(3 * rank * rank + rank) * 8; }

int cals_engine_create(cals_tensor* t, int r_star, int n_models, const int32_t* ranks,
                       int trace_capacity, cals_engine** out) {
  CALS_CHECK(t && out, kErrInvalid, "null argument");
  { const int rc_ = check_current_device(*t->t); if (rc_) return rc_; }
  Engine* e = nullptr;
  int rc = engine_create(t->t, r_star, n_models, ranks, trace_capacity, &e);
  if (rc) return rc;
  *out = new cals_engine{e};
  return kOk;
}

int cals_engine_destroy(cals_engine* e) {
  if (e) {
    engine_free(e->e);
    delete e;
  }
  return kOk;
}

int cals_engine_pool(cals_engine* e, double** pool, int64_t* elems) {
  CALS_CHECK(e, kErrInvalid, "null engine");
  if (pool) *pool = e->e->h_st.pool;
  if (elems) *elems = e->e->pool_elems;
  return kOk;
}

int cals_engine_load_pool(cals_engine* e, const double* src, int src_is_device, void* stream) {
  CALS_CHECK(e && src, kErrInvalid, "null argument");
  CALS_CUDA_TRY(cudaMemcpyAsync(e->e->h_st.pool, src, size_t(e->e->pool_elems) * 8,
                                src_is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                (cudaStream_t)stream));
  return kOk;
}

int cals_engine_run(cals_engine* e, double tol, int max_iterations, double sqnorm, int use_graph,
                    void* stream, int* iterations) {
  CALS_CHECK(e, kErrInvalid, "null engine");
  const int rc = engine_run(e->e, tol, max_iterations, sqnorm, use_graph, (cudaStream_t)stream,
                            iterations);
#ifdef CALS_UPD_PROFILE
  {
    static long long h[3][4096][13];
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(h, g_upd_prof, sizeof(h));
    const int ns = std::min(e->e->n_models, 4096);
    for (int n = 0; n < 3; ++n) {
      long long t0 = LLONG_MAX, t0max = 0, t1 = 0, cmax = 0, csum = 0;
      int cnt = 0;
      for (int sl = 0; sl < ns; ++sl) {
        const long long* p = h[n][sl];
        if (p[1] <= p[0]) continue;
        t0 = std::min(t0, p[0]); t0max = std::max(t0max, p[0]); t1 = std::max(t1, p[1]);
        cmax = std::max(cmax, p[2]); csum += p[2]; ++cnt;
      }
      fprintf(stderr, "[updprof] mode %d: span %lld ns, last block entry +%lld ns, block clk max %lld mean %lld\n",
              n, t1 - t0, t0max - t0, cmax, cnt ? csum / cnt : 0);
      // mean stamps (clk since entry): state copy, slot loads, H, chol+stage, solve+gram, pre-error
      long long ms[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
      for (int sl = 0; sl < ns; ++sl)
        for (int i = 0; i < 9; ++i) ms[i] += h[n][sl][4 + i];
      if (cnt)
        fprintf(stderr, "[updprof]   mean stamps: sst %lld, slot %lld, H %lld, chol+stage %lld, solve+gram %lld, pre-err %lld, end %lld\n",
                ms[0] / cnt, ms[1] / cnt, ms[2] / cnt, ms[3] / cnt, ms[4] / cnt, ms[5] / cnt, csum / cnt);
      if (cnt)
        fprintf(stderr, "[updprof]   inside solve+gram: solved %lld, written %lld, gram %lld\n",
                ms[6] / cnt, ms[7] / cnt, ms[8] / cnt);
    }
  }
#endif
  return rc;
}

int cals_engine_last_launches(cals_engine* e, long long* launches) {
  CALS_CHECK(e && launches, kErrInvalid, "null argument");
  *launches = e->e->last_launches;
  return kOk;
}

int cals_engine_pool_download(cals_engine* e, double* host_pool, void* stream) {
  CALS_CHECK(e && host_pool, kErrInvalid, "null engine or buffer");
  Engine* g = e->e;
  if (g->n_models == 0 || g->pool_elems == 0) return kOk;
  CALS_CUDA_TRY(cudaMemcpyAsync(host_pool, g->h_st.pool, size_t(g->pool_elems) * 8,
                                cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  return kOk;
}

int cals_engine_results(cals_engine* e, double* pool, int32_t* status, int32_t* iterations,
                        double* error, double* fit, int32_t* retire_seq, double* seconds_active,
                        double* lambdas, void* stream) {
  CALS_CHECK(e, kErrInvalid, "null engine");
  Engine* g = e->e;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t nm = size_t(g->n_models);
  if (nm == 0) return kOk;
  const EngState& h = g->h_st;
  // the small per-model arrays land in one page-locked block (async copies
  // are cheap there; pageable ones each cost a synchronous round trip), then
  // one host copy each into the caller's arrays
  const size_t lam_bytes = size_t(g->lam_elems) * 8;
  const size_t need = nm * (4 + 4 + 8 + 8 + 4 + 8 + 8) + lam_bytes + 64;
  if (g->h_results_bytes < need) {
    if (g->h_results) cudaFreeHost(g->h_results);
    g->h_results = nullptr;
    g->h_results_bytes = 0;
    CALS_CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&g->h_results), need, 0));
    g->h_results_bytes = need;
  }
  char* hb = g->h_results;
  int32_t* hs = reinterpret_cast<int32_t*>(hb);
  int32_t* hi = hs + nm;
  int32_t* hq = hi + nm;
  double* he = reinterpret_cast<double*>(hb + ((nm * 12 + 7) / 8) * 8);
  double* hf = he + nm;
  unsigned long long* ta = reinterpret_cast<unsigned long long*>(hf + nm);
  unsigned long long* tr = ta + nm;
  double* hl = reinterpret_cast<double*>(tr + nm);
  if (lambdas) {
    lambdas_kernel<<<std::min<int>(g->n_models, 1024), 32, 0, s>>>(g->d_st, g->d_lam_off,
                                                                 g->d_lam);
    CALS_CUDA_TRY(cudaGetLastError());
    CALS_CUDA_TRY(cudaMemcpyAsync(hl, g->d_lam, lam_bytes, cudaMemcpyDeviceToHost, s));
  }
  if (pool)
    CALS_CUDA_TRY(cudaMemcpyAsync(pool, h.pool, size_t(g->pool_elems) * 8, cudaMemcpyDeviceToHost, s));
  if (status) CALS_CUDA_TRY(cudaMemcpyAsync(hs, h.status, nm * 4, cudaMemcpyDeviceToHost, s));
  if (iterations) CALS_CUDA_TRY(cudaMemcpyAsync(hi, h.iters, nm * 4, cudaMemcpyDeviceToHost, s));
  if (retire_seq)
    CALS_CUDA_TRY(cudaMemcpyAsync(hq, h.retire_seq, nm * 4, cudaMemcpyDeviceToHost, s));
  if (error) CALS_CUDA_TRY(cudaMemcpyAsync(he, h.err, nm * 8, cudaMemcpyDeviceToHost, s));
  if (fit) CALS_CUDA_TRY(cudaMemcpyAsync(hf, h.fit, nm * 8, cudaMemcpyDeviceToHost, s));
  if (seconds_active) {
    CALS_CUDA_TRY(cudaMemcpyAsync(ta, h.t_admit, nm * 8, cudaMemcpyDeviceToHost, s));
    CALS_CUDA_TRY(cudaMemcpyAsync(tr, h.t_retire, nm * 8, cudaMemcpyDeviceToHost, s));
  }
  CALS_CUDA_TRY(cudaStreamSynchronize(s));
  if (status) memcpy(status, hs, nm * 4);
  if (iterations) memcpy(iterations, hi, nm * 4);
  if (retire_seq) memcpy(retire_seq, hq, nm * 4);
  if (error) memcpy(error, he, nm * 8);
  if (fit) memcpy(fit, hf, nm * 8);
  if (lambdas) memcpy(lambdas, hl, lam_bytes);
  if (seconds_active)
    for (size_t k = 0; k < nm; ++k) seconds_active[k] = (double)(tr[k] - ta[k]) * 1e-9;
  return kOk;
}

int cals_engine_trace(cals_engine* e, int32_t* widths, int32_t* n_active, double* seconds,
                      int capacity, int* count) {
  CALS_CHECK(e && count, kErrInvalid, "null argument");
  Engine* g = e->e;
  int plans = 0;
  CALS_CUDA_TRY(cudaMemcpy(&plans, &g->d_st->plans_done, 4, cudaMemcpyDeviceToHost));
  const int recs = std::min(plans, g->trace_cap);
  const int iters = std::max(0, recs - 1);
  *count = iters;
  if (iters == 0 || capacity <= 0) return kOk;
  std::vector<int> w(recs), a(recs);
  std::vector<unsigned long long> tt(recs);
  CALS_CUDA_TRY(cudaMemcpy(w.data(), g->h_st.tr_width, recs * 4, cudaMemcpyDeviceToHost));
  CALS_CUDA_TRY(cudaMemcpy(a.data(), g->h_st.tr_active, recs * 4, cudaMemcpyDeviceToHost));
  CALS_CUDA_TRY(cudaMemcpy(tt.data(), g->h_st.tr_time, recs * 8, cudaMemcpyDeviceToHost));
  for (int i = 0; i < std::min(iters, capacity); ++i) {
    if (widths) widths[i] = w[i];
    if (n_active) n_active[i] = a[i];
    if (seconds) seconds[i] = (double)(tt[i + 1] - tt[i]) * 1e-9;
  }
  return kOk;
}

int cals_engine_set_tensor(cals_engine* e, cals_tensor* t) {
  CALS_CHECK(e && t, kErrInvalid, "null argument");
  Engine* g = e->e;
  CALS_CHECK(t->t->order == g->order, kErrInvalid, "tensor order differs from the engine's");
  { const int rc_ = check_current_device(*t->t); if (rc_) return rc_; }
  CALS_CHECK(t->t->device == g->device, kErrInvalid,
             "tensor lives on another CUDA device than the engine");
  // the previously bound tensor may already be destroyed: compare against the
  // engine's own copy of the dims and the tensor's unique id, never the pointer
  for (int n = 0; n < g->order; ++n)
    CALS_CHECK(t->t->dims[n] == g->h_st.dims[n], kErrInvalid,
               "tensor dims differ from the engine's");
  if (t->t->uid != g->tensor_uid) {
    g->t = t->t;
    g->tensor_uid = t->t->uid;
    // the captured graph embeds the old tensor's TMA descriptors (and Ozaki
    // slices): re-captured at the next run and swapped into the executable
    // graph by cudaGraphExecUpdate (same topology, new kernel parameters)
    g->graph_stale = true;
  }
  return kOk;
}

int cals_nnls_rows(int rows, int rank, const double* m, int64_t ldm, const double* h,
                   uint32_t* active, double* x, int64_t ldx, int32_t* converged, int max_iter,
                   void* stream) {
  CALS_CHECK(rows >= 0 && rank >= 1 && rank <= kFastR, kErrInvalid,
             "rank must be in [1, 32] for the NNLS kernel");
  CALS_CHECK(m && h && active && x && converged, kErrInvalid, "null argument");
  if (rows == 0) return kOk;
  const int warps = 4;
  const size_t smem = (size_t(rank) * rank + size_t(warps) * kNnlsWs) * 8;
  CALS_CUDA_TRY(raise_smem_limit((const void*)nnls_rows_kernel, smem));
  const int blocks = std::max(1, std::min((rows + warps - 1) / warps, 148 * 8));
  nnls_rows_kernel<<<blocks, 32 * warps, smem, (cudaStream_t)stream>>>(
      rows, rank, m, ldm, h, active, x, ldx, converged, max_iter);
  CALS_CUDA_TRY(cudaGetLastError());
  return kOk;
}

int cals_engine_prepare(cals_engine* e, void* stream) {
  CALS_CHECK(e, kErrInvalid, "null engine");
  return engine_prepare_slices(e->e, (cudaStream_t)stream, false);
}

int cals_engine_set_nonneg(cals_engine* e, int enabled) {
  CALS_CHECK(e, kErrInvalid, "null engine");
  return engine_set_nonneg(e->e, enabled);
}

int cals_engine_nnls_warnings(cals_engine* e, int32_t* flags) {
  CALS_CHECK(e && flags, kErrInvalid, "null argument");
  Engine* g = e->e;
  if (!g->h_st.nnls_warn || g->n_models == 0) {
    for (int k = 0; k < g->n_models; ++k) flags[k] = 0;
    return kOk;
  }
  CALS_CUDA_TRY(cudaMemcpy(flags, g->h_st.nnls_warn, size_t(g->n_models) * 4,
                           cudaMemcpyDeviceToHost));
  return kOk;
}

int cals_engine_update_failures(cals_engine* e, int32_t* flags) {
  CALS_CHECK(e && flags, kErrInvalid, "null argument");
  Engine* g = e->e;
  if (g->n_models == 0) return kOk;
  CALS_CUDA_TRY(cudaMemcpy(flags, g->h_st.failed, size_t(g->n_models) * 4,
                           cudaMemcpyDeviceToHost));
  return kOk;
}

int cals_engine_set_line_search(cals_engine* e, int enabled, double alpha) {
  CALS_CHECK(e, kErrInvalid, "null engine");
  CALS_CHECK(!enabled || alpha <= 0.0 || alpha > 1.0, kErrInvalid,
             "extrapolation alpha must be > 1 (or <= 0 for the i^(1/3) rule)");
  return engine_set_line_search(e->e, enabled, alpha);
}

// ---- step-wise driving (host-orchestrated loops, e.g. the mode-0-sharded
// configuration with an all-reduce between the MTTKRP and the update) ------
int cals_engine_begin(cals_engine* e, double tol, int max_iterations, double sqnorm,
                      void* stream) {
  CALS_CHECK(e, kErrInvalid, "null engine");
  CALS_CHECK(max_iterations >= 1, kErrInvalid, "max_iterations must be >= 1");
  CALS_CHECK(sqnorm > 0.0, kErrInvalid, "tensor squared norm must be positive");
  Engine* g = e->e;
  CALS_CHECK(!g->h_st.ls_enabled, kErrUnsupported,
             "line search is not supported by the step-wise (sharded) driver");
  cudaStream_t s = (cudaStream_t)stream;
  // the previous step-wise run may still be in flight on this stream
  CALS_CUDA_TRY(cudaStreamSynchronize(s));
  int rc = engine_reset(g, tol, max_iterations, sqnorm, s);
  if (rc) return rc;
  if (g->n_models == 0) {
    *g->h_done = 1;
    return kOk;
  }
  rc = engine_prepare_slices(g, s);
  if (rc) return rc;
  // the step-wise driver reduces partial MTTKRPs between the calls: no fusion
  g->lo_target = -1;
  g->lo_carry = false;
  g->ua.lo[0].src = -1;
  g->ua.lo[1].src = -1;
  return enqueue_plan(g, s);  // initial admission
}

int cals_engine_enqueue_mttkrp(cals_engine* e, int mode, void* stream) {
  CALS_CHECK(e && mode >= 0 && mode < e->e->order, kErrInvalid, "bad argument");
  return enqueue_mode_mttkrp(e->e, mode, (cudaStream_t)stream);
}

int cals_engine_enqueue_update(cals_engine* e, int mode, void* stream) {
  CALS_CHECK(e && mode >= 0 && mode < e->e->order, kErrInvalid, "bad argument");
  return enqueue_mode_update(e->e, mode, (cudaStream_t)stream);
}

int cals_engine_enqueue_plan(cals_engine* e, void* stream) {
  CALS_CHECK(e, kErrInvalid, "null engine");
  return enqueue_plan(e->e, (cudaStream_t)stream);
}

int cals_engine_done(cals_engine* e, int* done) {
  CALS_CHECK(e && done, kErrInvalid, "null argument");
  *done = *(volatile int*)e->e->h_done;
  return kOk;
}

int cals_engine_buffers(cals_engine* e, double** mttkrp_out, double** grams, int64_t* ld,
                        int64_t* gram_stride, double** factors) {
  CALS_CHECK(e, kErrInvalid, "null engine");
  Engine* g = e->e;
  if (mttkrp_out) *mttkrp_out = g->h_st.Mout;
  if (grams) *grams = g->h_st.grams;
  if (ld) *ld = g->ld;
  if (gram_stride) *gram_stride = g->gram_stride;
  if (factors)
    for (int n = 0; n < g->order; ++n) factors[n] = g->h_st.F[n];
  return kOk;
}

int cals_engine_variant(cals_engine* e, int mode, int* variant, int* bm, int* bn, int* splits) {
  CALS_CHECK(e && mode >= 0 && mode < e->e->order, kErrInvalid, "bad argument");
  const int v = e->e->variants[mode];
  if (variant) *variant = v;
  if (bm) *bm = variant_info(v).BM;
  if (bn) *bn = variant_info(v).BN;
  if (splits) *splits = e->e->t->plans[mode].S;
  return kOk;
}

}  // extern "C"
