// Split per-model update (ranks <= 32, Cholesky / pinv updates): the work of
// als.py:74-96 + driver.py:213-235 divided by what the next fused MTTKRP
// actually waits for.
//
//   prep(n)  -- OFF the critical path, on a side stream concurrently with the
//               fused MTTKRP of mode n: the Hadamard of the other modes'
//               Gramians (ascending, driver.py:223-225), the finite check on
//               H and the upper Cholesky of H (dpotrf), or the eigen
//               pseudo-inverse when H admits none (als.py:86-96); at n = 0
//               also the Gramians of freshly admitted models
//               (driver.py:203-205).  H_n needs no M_n, so none of this waits
//               for the contraction.  One warp per model: it shares the SM
//               with the contraction's CTA.
//   solve(n) -- ON the critical path, right after the MTTKRP: one CTA per
//               (model, 256-row chunk; one chunk at every benchmarked shape)
//               solves its rows A = M H^-1 (dpotrs order) or A = M pinv(H),
//               all-or-nothing on a non-finite M block (ValueError -> FAILED,
//               als.py:84-85), and refreshes G_n from the solved rows still in
//               shared memory (driver.py:234).  The last mode also finishes
//               the fast error, the fit and the stopping rule (als.py:99-124,
//               driver.py:241-273).  With several chunks, the chunk that
//               arrives last sums the per-chunk partial Gramians (fixed
//               order).  A non-finite Cholesky solution (the reference then
//               redoes the block with the pinv, als.py:88-90) is redone by
//               that chunk too (cold path).
//
// Results are independent of the slot a model occupies and of the other
// models (fixed per-model reduction orders), so CALS == SEQUENTIAL bitwise.
#pragma once

#include "engine_state.cuh"

namespace cals {

constexpr int kSolveRows = 256;  // rows (threads) per solve CTA
constexpr int kPrepThreads = 32;  // one warp per model

// prep / solve status of a model for the current mode
enum PrepFlag : int { kPrepChol = 0, kPrepPinv = 1, kPrepBadH = 2, kPrepFailed = 3 };

struct UpdArgs {
  EngState* st;            // decide_model (last mode), scalars
  const int* n_active;     // &st->n_active (device)
  const int4* slot_info;   // {model, rank, column offset, Gramian offset}
  int* failed;
  int* fresh;
  int* pflag;              // per model, PrepFlag for the current mode
  int* arrive;             // per model arrival counter of the solve chunks
  int* solbad;             // per model: a Cholesky solution entry was non-finite
  double* grams;           // [order][gram_stride]
  long long gram_stride;
  double* ubuf;            // per model 3 R x R blocks: U strictly upper with
                           // 1/U[a][a] on the diagonal (kPrepChol) or pinv(H)
                           // (kPrepPinv); U^T; H (Hadamard of the others)
  double* gpart;           // per model [chunk][R][R] partial Gramians (chunks > 1)
  double* ipart;           // last mode: per model [chunk] partial <A, M>
  const double* Mout;
  // M_n as split-K partials (SplitDefer, internal.h) instead of Mout: set per
  // solve launch of a non-last mode whose contraction skipped its reduction
  // (mS <= 1: read Mout)
  const double* mpart;
  long long mpart_stride;
  long long mpart_ld;
  int mS;
  double* F[kMaxOrder];
  long long dims[kMaxOrder];
  long long ld;
  int order;
  // Lo-slice fusion: the solve of mode lo[t].src (-1: none) also writes the
  // Ozaki Lo slices of its factor columns for a later INT8 contraction that
  // takes F[src] as its Lo operand (the oz_slice_cols* arithmetic).  Target 0
  // is consumed in the same driver iteration (that contraction skips its
  // slicing kernel); target 1 by the next iteration's mode-0 contraction,
  // whose slicing kernel only runs when the plan changed the column layout
  // in between (*lo_stale, set by the plan kernel, cleared here).
  // OzLoLayout in internal.h.
  struct LoTarget {
    uint8_t* ls;
    int* cex;
    int* queue;           // the contraction's unit counter (target 0 zeroes it)
    long long stride;     // cap_pad * Kp
    int Kp;
    int Dp;
    int src;
  } lo[2];
  int* lo_stale;
  int rev;  // solve CTAs take the active slots last-first (upd_solve_kernel)
};

// Shared memory of upd_solve_kernel<RB> (SolveSmem in update2.cu):
// U, U^T (pitch RB + 1), H and G (RB x RB), 1/diag, the kSolveRows x (RB + 1)
// row tile, 8 x 64 Gram partials, reduction scratch
__host__ __device__ constexpr size_t solve_smem_bytes(int RB) {
  return size_t(2 * RB * (RB + 1) + 2 * RB * RB + RB + (RB & 1) + kSolveRows * (RB + 1) + 8 * 64 +
                32 + RB) * 8 + 16;
}

using PrepKernel = void (*)(UpdArgs, int);
using SolveKernel = void (*)(UpdArgs, int, int);
// kernels of rank bucket rb (8 / 16 / 24 / 32) and the solve kernels' dynamic
// shared memory
void split_kernels_for(int rb, PrepKernel* prep, SolveKernel* solve, SolveKernel* last,
                       size_t* smem);

}  // namespace cals
