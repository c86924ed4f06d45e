// Split per-model update kernels (design: update2.cuh).
#include "update.cuh"
#include "update2.cuh"
#include "ozaki.cuh"

namespace cals {

#ifdef CALS_SOLVE_PROFILE
// per (mode, CTA) clock64 stamps of the solve kernel: [0] R, [1..8] phases
__device__ long long g_solve_prof[8][2048][16];
#define SOLVE_STAMP(i) \
  if (tid == 0 && blockIdx.x < 2048) g_solve_prof[n][blockIdx.x][i] = clock64() - t_entry;
#else
#define SOLVE_STAMP(i)
#endif

// G = A^T A of the column block A[i][r] (rows x R, row stride ld) by one warp
// (fresh admissions only).  32-row chunks: lane i loads row i of the next
// chunk into registers while the warp accumulates the current chunk from
// shared memory (pitch P odd); each lane owns (a, b) pairs summed over
// ascending rows (one chain per pair, as block_gram_fast); upper mirrored.
template <int RB>
__device__ __forceinline__ void warp_gram(const double* __restrict__ A, long long ld, int rows,
                                          int R, double* __restrict__ T, double* __restrict__ G) {
  constexpr int NP = (RB * (RB + 1) / 2 + 31) / 32;
  const int lane = threadIdx.x & 31;
  const int P = fast_pitch(R);
  const int npairs = R * (R + 1) / 2;
  int pab[NP];  // a | b << 8, -1 past the pairs
  double acc[NP];
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    const int p = lane + 32 * j;
    acc[j] = 0.0;
    pab[j] = -1;
    if (p < npairs) {
      int aa = 0, rem = p;
      while (rem >= R - aa) {
        rem -= R - aa;
        ++aa;
      }
      pab[j] = aa | ((aa + rem) << 8);
    }
  }
  double v[RB];
  auto load_row = [&](int i) {
#pragma unroll
    for (int c = 0; c < RB; ++c) v[c] = (i < rows && c < R) ? A[(long long)i * ld + c] : 0.0;
  };
  load_row(lane);
  for (int base = 0; base < rows; base += 32) {
    const int cnt = min(32, rows - base);
    __syncwarp();  // the previous chunk's reads of T are done
#pragma unroll
    for (int c = 0; c < RB; ++c)
      if (c < R) T[lane * P + c] = v[c];
    __syncwarp();
    if (base + 32 < rows) load_row(base + 32 + lane);  // in flight during the sums
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      if (pab[j] < 0) continue;
      const double* xa = T + (pab[j] & 255);
      const double* xb = T + (pab[j] >> 8);
      double s = acc[j];
      int r = 0;
      for (; r + 4 <= cnt; r += 4) {
        const double x0 = xa[r * P], y0 = xb[r * P], x1 = xa[(r + 1) * P], y1 = xb[(r + 1) * P];
        const double x2 = xa[(r + 2) * P], y2 = xb[(r + 2) * P], x3 = xa[(r + 3) * P],
                     y3 = xb[(r + 3) * P];
        s = fma(x0, y0, s);
        s = fma(x1, y1, s);
        s = fma(x2, y2, s);
        s = fma(x3, y3, s);
      }
      for (; r < cnt; ++r) s = fma(xa[r * P], xb[r * P], s);
      acc[j] = s;
    }
  }
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    if (pab[j] < 0) continue;
    const int aa = pab[j] & 255, bb = pab[j] >> 8;
    G[aa * R + bb] = acc[j];
    G[bb * R + aa] = acc[j];
  }
}

// H = Hadamard of the Gramians of every mode but n (ascending), R x R, into
// shared memory; returns whether any entry this thread formed is non-finite.
__device__ __forceinline__ int hadamard_others(const double* grams, long long gs, long long go,
                                               int N, int n, int R, double* H, int t0, int nt) {
  int bad = 0;
  for (int idx = t0; idx < R * R; idx += nt) {
    double h = 1.0;
    bool first = true;
    for (int i = 0; i < N; ++i) {
      if (i == n) continue;
      const double g = grams[i * gs + go + idx];
      h = first ? g : h * g;
      first = false;
    }
    H[idx] = h;
    bad |= !isfinite(h);
  }
  return bad;
}

template <int RB>
__global__ void __launch_bounds__(kPrepThreads, 16) upd_prep_kernel(UpdArgs a, int n) {
  __shared__ __align__(16) double H[RB * RB];
  __shared__ __align__(16) double T[32 * (RB + 1)];  // Gram staging; V of the pinv
  __shared__ double lam[RB];
  __shared__ double invd[RB];
  __shared__ int flag;
  const int lane = threadIdx.x;
  const int slot = blockIdx.x;
  const int na = *a.n_active;
  const int4 si = a.slot_info[slot];  // slot < max_slots: in bounds
  if (slot >= na) return;
  const int k = si.x, R = si.y, off = si.z;
  const long long go = si.w;
  const int N = a.order;
  if (a.failed[k]) {
    if (lane == 0) a.pflag[k] = kPrepFailed;
    return;
  }
  const long long gs = a.gram_stride;
  if (n == 0 && a.fresh[k]) {  // Gramians of the admitted starting point (driver.py:203-205)
    for (int i = 1; i < N; ++i)
      warp_gram<RB>(a.F[i] + off, a.ld, (int)a.dims[i], R, T, a.grams + i * gs + go);
    if (lane == 0) a.fresh[k] = 0;
    __syncwarp();
  }
  const int bad = __any_sync(0xffffffffu, hadamard_others(a.grams, gs, go, N, n, R, H, lane, 32));
  if (bad) {  // non-finite h: update_factor raises (als.py:84-85)
    if (lane == 0) a.pflag[k] = kPrepBadH;
    return;
  }
  __syncwarp();
  // per model: [U | U^T | H] (3 R x R blocks); H feeds the last mode's fast
  // error (sum of H o G_{N-1}) without reloading the other Gramians
  double* U = a.ubuf + 3 * go;
  double* V = U + R * R;
  for (int idx = lane; idx < R * R; idx += 32) V[R * R + idx] = H[idx];
  warp_cholesky_rb<RB>(H, R, invd, &flag);
  __syncwarp();
  if (flag) {
    for (int idx = lane; idx < R * R; idx += 32) {
      const int r = idx / R, c = idx - r * R;
      const double u = r < c ? H[idx] : (r == c ? invd[r] : 0.0);
      U[idx] = u;            // U[r][c] (strictly upper), 1/U[r][r] on the diagonal
      V[c * R + r] = u;      // U^T: the back substitution reads rows of it
    }
    if (lane == 0) a.pflag[k] = kPrepChol;
  } else {  // dpotrf failed: pinv(H) (als.py:91-96)
    hadamard_others(a.grams, gs, go, N, n, R, H, lane, 32);
    __syncwarp();
    block_pinv(H, T, lam, R);
    for (int idx = lane; idx < R * R; idx += 32) U[idx] = H[idx];
    if (lane == 0) a.pflag[k] = kPrepPinv;
  }
}

// x <- m P for one shared-memory row (als.py:96: m @ pinv), b ascending as
// block_apply_pinv
template <int RB>
__device__ __forceinline__ void apply_pinv_row(double* __restrict__ xs, const double* __restrict__ P,
                                               int R) {
  double m[RB];
#pragma unroll
  for (int b = 0; b < RB; ++b) m[b] = b < R ? xs[b] : 0.0;
  for (int c = 0; c < R; ++c) {
    double s = 0.0;
#pragma unroll
    for (int b = 0; b < RB; ++b)
      if (b < R) s = fma(m[b], P[b * R + c], s);
    xs[c] = s;
  }
}

// the last mode's error / fit / stopping rule with the scalars loaded at
// kernel entry (thread 0): only stores left on the critical path
__device__ __forceinline__ void finish_model_pre(const UpdArgs& a, int k, double msq, double inner,
                                                 const DecideIn& d, int ls_on) {
  EngState* st = a.st;
  st->iters[k] = d.it;
  double e = d.sqnorm + msq - 2.0 * inner;
  e = e > 0.0 ? e : 0.0;  // als.py:114-115 (NaN clamps to 0 as there)
  if (ls_on)
    st->e_tmp[k] = e;  // decided after the line-search candidate (ls_finish)
  else
    decide_model_with(st, k, e, d);
}

// the last mode's error / fit / stopping rule from the summed pieces
__device__ __forceinline__ void finish_model(const UpdArgs& a, int k, double msq, double inner,
                                             bool updated) {
  // scalars that change between runs / line-search switches are read from
  // the device state, never baked into a captured graph
  EngState* st = a.st;
  ++st->iters[k];
  const double sq = st->sqnorm;
  double e = updated ? sq + msq - 2.0 * inner : sq;
  e = e > 0.0 ? e : 0.0;  // als.py:114-115 (NaN clamps to 0 as there)
  if (st->ls_enabled)
    st->e_tmp[k] = e;  // decided after the line-search candidate (ls_finish)
  else
    decide_model(st, k, e);
}

// One factor row: A = M H^-1 with H = U^T U (dpotrs: forward substitution
// with U^T, then back substitution with U; reciprocal diagonal).  The k loops
// stay rolled: the row lives in registers and shifts down one slot per step
// (register rotation), so every step reads its operands at static indices.
// Us / Vs hold U and U^T pre-shifted by the solve kernel: Us[k][j] =
// U[k][k+1+j], Vs[k][j] = U^T[k][k-1-j], zero past the triangle.  Each
// element sees exactly the unrolled dtrsm sequence x_c = fma(-u, y_k, x_c),
// k ascending (forward) / descending (back); the slots past the triangle only
// carry unused values.  A fully unrolled per-rank solve is ~R^2 instructions
// of straight-line code fetched cold by every CTA (ncu: no_instruction was the
// top stall); this body is ~6 R instructions.
// One substitution sweep for R <= 16 with the next step's pre-shifted row and
// reciprocal diagonal loaded while the current step runs (two register
// buffers, steps taken in pairs): a step then costs one DMUL + one DFMA of
// latency instead of two dependent shared-memory round trips on top.  The FMA
// sequence per element is solve_row_exact's.  `dir` +1: forward (k = 0 ..
// R-1, W = Us), -1: back (k = R-1 .. 0, W = Vs).
template <int R>
__device__ __forceinline__ void subst_pipelined(double (&r)[R], double* __restrict__ xs,
                                                const double* __restrict__ W,
                                                const double* __restrict__ invd, int dir) {
  constexpr int RS = R + (R & 1);
  constexpr int RM = R > 1 ? R - 1 : 1;
  double ua[RM], ub[RM], da, db;
  auto load = [&](double (&u)[RM], double& d, int s) {  // s: step index 0 .. R-1
    const int k = dir > 0 ? s : R - 1 - s;
    d = invd[k];
    // 16-byte loads (rows of RS doubles, RS even, 16-byte aligned): half the
    // shared-memory instructions of the step, which all warps issue
    const double2* w2 = reinterpret_cast<const double2*>(W + k * RS);
#pragma unroll
    for (int j = 0; j + 1 < R; j += 2) {
      const double2 p = w2[j >> 1];
      u[j] = p.x;
      if (j + 1 < RM) u[j + 1] = p.y;
    }
  };
  auto step = [&](const double (&u)[RM], double d, int s) {
    const int k = dir > 0 ? s : R - 1 - s;
    const double y = r[0] * d;
    xs[k] = y;
#pragma unroll
    for (int j = 0; j + 1 < R; ++j) r[j] = fma(-u[j], y, r[j + 1]);
  };
  load(ua, da, 0);
  int s = 0;
#pragma unroll 1
  for (; s + 1 < R; s += 2) {
    load(ub, db, s + 1);
    step(ua, da, s);
    load(ua, da, s + 2 < R ? s + 2 : R - 1);
    step(ub, db, s + 1);
  }
  if (s < R) step(ua, da, s);
}

template <int R>
__device__ __forceinline__ void solve_row_exact(double* __restrict__ xs,
                                                const double* __restrict__ Us,
                                                const double* __restrict__ Vs,
                                                const double* __restrict__ invd) {
  constexpr int RS = R + (R & 1);
  double r[R];
#pragma unroll
  for (int c = 0; c < R; ++c) r[c] = xs[c];
  if constexpr (R <= 16) {
    subst_pipelined<R>(r, xs, Us, invd, 1);
#pragma unroll
    for (int j = 0; j < R; ++j) r[j] = xs[R - 1 - j];
    subst_pipelined<R>(r, xs, Vs, invd, -1);
  } else {
#pragma unroll 1
    for (int k = 0; k < R; ++k) {
      const double yk = r[0] * invd[k];
      xs[k] = yk;
      const double2* u = reinterpret_cast<const double2*>(Us + k * RS);  // 16-byte loads
#pragma unroll
      for (int j = 0; j + 1 < R; j += 2) {
        const double2 p = u[j >> 1];
        r[j] = fma(-p.x, yk, r[j + 1]);
        if (j + 2 < R) r[j + 1] = fma(-p.y, yk, r[j + 2]);
      }
    }
#pragma unroll
    for (int j = 0; j < R; ++j) r[j] = xs[R - 1 - j];
#pragma unroll 1
    for (int k = R - 1; k >= 0; --k) {
      const double xk = r[0] * invd[k];
      xs[k] = xk;
      const double2* v = reinterpret_cast<const double2*>(Vs + k * RS);
#pragma unroll
      for (int j = 0; j + 1 < R; j += 2) {
        const double2 p = v[j >> 1];
        r[j] = fma(-p.x, xk, r[j + 1]);
        if (j + 2 < R) r[j + 1] = fma(-p.y, xk, r[j + 2]);
      }
    }
  }
}

template <int RB, int R = 1>
__device__ __forceinline__ void solve_row_dispatch(int r, double* xs, const double* U,
                                                   const double* V, const double* invd) {
  if constexpr (R <= RB) {
    if (r == R)
      solve_row_exact<R>(xs, U, V, invd);
    else
      solve_row_dispatch<RB, R + 1>(r, xs, U, V, invd);
  }
}

// Gramian X^T X of the rows [0, cnt) of the tile X (pitch P, R columns) on
// the FP64 tensor cores (DMMA.8x8x4): 8 x 8 output tiles of the upper tile
// triangle; with few tiles the rows are split into up to 8 / tiles parts
// (one warp each) whose partial tiles are added in part order through
// `scr` (>= 8 * 64 doubles).  Result (full symmetric) in Gs (R x R, smem).
__device__ __forceinline__ void tile_gram_tc(const double* __restrict__ X, int P, int cnt, int R,
                                             double* __restrict__ scr, double* __restrict__ Gs) {
  constexpr int kWarps = kSolveRows / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int T = (R + 7) >> 3;
  const int ntiles = T * (T + 1) / 2;
  const int parts = ntiles >= kWarps ? 1 : kWarps / ntiles;
  const int r_lo = lane >> 2, k_lo = lane & 3;
  const int steps = (cnt + 3) >> 2;  // K steps of 4 rows
  for (int task = warp; task < ntiles * parts; task += kWarps) {
    const int t = task / parts, part = task - t * parts;
    int ti = 0, rem = t;
    while (rem >= T - ti) {
      rem -= T - ti;
      ++ti;
    }
    const int tj = ti + rem;
    const int ca = ti * 8 + r_lo, cb = tj * 8 + r_lo;
    const bool va = ca < R, vb = cb < R;
    const int s0 = steps * part / parts, s1 = steps * (part + 1) / parts;
    // two independent DMMA chains (even / odd K steps), added at the end:
    // half the dependent-accumulation latency of one chain
    double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
    int st = s0;
    for (; st + 2 <= s1; st += 2) {
      const int kk = st * 4 + k_lo, kn = kk + 4;
      const bool vk = kk < cnt, vn = kn < cnt;
      const double av = (va && vk) ? X[kk * P + ca] : 0.0;
      const double bv = (vb && vk) ? X[kk * P + cb] : 0.0;
      const double an = (va && vn) ? X[kn * P + ca] : 0.0;
      const double bn = (vb && vn) ? X[kn * P + cb] : 0.0;
      dmma_8x8x4(d0, d1, av, bv);
      dmma_8x8x4(e0, e1, an, bn);
    }
    if (st < s1) {
      const int kk = st * 4 + k_lo;
      const bool vk = kk < cnt;
      const double av = (va && vk) ? X[kk * P + ca] : 0.0;
      const double bv = (vb && vk) ? X[kk * P + cb] : 0.0;
      dmma_8x8x4(d0, d1, av, bv);
    }
    d0 += e0;
    d1 += e1;
    if (parts == 1) {
      const int gr = ti * 8 + r_lo, gc = tj * 8 + 2 * k_lo;
      if (gr < R && gc < R) {
        Gs[gr * R + gc] = d0;
        Gs[gc * R + gr] = d0;
      }
      if (gr < R && gc + 1 < R) {
        Gs[gr * R + gc + 1] = d1;
        Gs[(gc + 1) * R + gr] = d1;
      }
    } else {
      scr[task * 64 + 2 * lane] = d0;
      scr[task * 64 + 2 * lane + 1] = d1;
    }
  }
  if (parts > 1) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < ntiles * 64; idx += kSolveRows) {
      const int t = idx >> 6, e = idx & 63;
      double s = scr[(t * parts) * 64 + e];
      for (int p = 1; p < parts; ++p) s += scr[(t * parts + p) * 64 + e];
      int ti = 0, rem = t;
      while (rem >= T - ti) {
        rem -= T - ti;
        ++ti;
      }
      const int tj = ti + rem;
      const int ln = e >> 1;  // lane that held the entry
      const int gr = ti * 8 + (ln >> 2), gc = tj * 8 + 2 * (ln & 3) + (e & 1);
      if (gr < R && gc < R) {
        Gs[gr * R + gc] = s;
        Gs[gc * R + gr] = s;
      }
    }
  }
}

// Lo-slice fusion (UpdArgs::lo_src): the Ozaki Lo slices of this model's
// columns [off, off + R) of F[n] -- every row, so only single-chunk solves --
// exactly as oz_slice_cols_kernel / oz_slice_cols_all_kernel form them: the
// column maximum over the Dp rows (scale_exp_checked), slice7 per element,
// zeros for p in [Dp, Kp).  A / ld: the factor block -- the solved rows still
// in shared memory, or (failure / pinv-redo paths) F[n] in global memory
// (this CTA's own stores, visible after the barrier that precedes the call).
// The target's fields come by value: taking the address of the kernel
// parameter block would make the compiler copy all of it to the stack at
// every solve CTA's entry.
__device__ __noinline__ void slice_lo_columns(uint8_t* __restrict__ ls, int* __restrict__ cex,
                                              int* queue, long long stride, int Kp, int Dp,
                                              int off, int R, const double* __restrict__ A,
                                              long long ld) {
  __shared__ int ex_s[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (queue && blockIdx.x == 0 && tid == 0) *queue = 0;  // the contraction's unit counter
  for (int c = warp; c < R; c += kSolveRows / 32) {
    double mx = 0.0;
#pragma unroll 4
    for (int p = lane; p < Dp; p += 32) mx = fmax(mx, oz::abs_or_inf(A[(long long)p * ld + c]));
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) {
      const int e = oz::scale_exp_checked(mx);
      ex_s[c] = e;
      cex[off + c] = e;
    }
  }
  __syncthreads();
  const int groups = Kp >> 2;  // 4 consecutive p per thread: one 32-bit word per slice
  for (int idx = tid; idx < R * groups; idx += kSolveRows) {
    const int c = idx / groups, p0 = (idx - c * groups) * 4;
    uint32_t w[oz::kSlices];
#pragma unroll
    for (int s = 0; s < oz::kSlices; ++s) w[s] = 0u;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int p = p0 + u;
      const double v = p < Dp ? A[(long long)p * ld + c] : 0.0;
      uint8_t sl[oz::kSlices];
      oz::slice7(v, ex_s[c], sl);
#pragma unroll
      for (int s = 0; s < oz::kSlices; ++s) w[s] |= uint32_t(sl[s]) << (8 * u);
    }
    uint8_t* dst = ls + size_t(off + c) * Kp + p0;
#pragma unroll
    for (int s = 0; s < oz::kSlices; ++s)
      *reinterpret_cast<uint32_t*>(dst + size_t(s) * stride) = w[s];
  }
}

// Every fusion target fed by the solve of mode n (UpdArgs::lo); block-uniform.
__device__ __forceinline__ void slice_lo_targets(const UpdArgs& a, int n, int off, int R,
                                                 const double* A, long long ld) {
#pragma unroll
  for (int t = 0; t < 2; ++t)
    if (a.lo[t].src == n) {
      slice_lo_columns(a.lo[t].ls, a.lo[t].cex, a.lo[t].queue, a.lo[t].stride, a.lo[t].Kp,
                       a.lo[t].Dp, off, R, A, ld);
      if (t == 1 && blockIdx.x == 0 && threadIdx.x == 0) *a.lo_stale = 0;
    }
}

// arr[n] for a runtime n without indexing the kernel parameter block (a
// dynamic index makes the compiler copy the array to the stack)
template <class T>
__device__ __forceinline__ T param_at(const T (&arr)[kMaxOrder], int n) {
  T v = arr[0];
#pragma unroll
  for (int i = 1; i < kMaxOrder; ++i)
    if (i == n) v = arr[i];
  return v;
}

// Shared-memory layout of upd_solve_kernel<RB> (doubles)
struct SolveSmem {
  int U, V, H, G, invd, X, scr, red, lam, total;
  __host__ __device__ constexpr SolveSmem(int RB)
      : U(0), V(RB * (RB + 1)), H(2 * RB * (RB + 1)), G(2 * RB * (RB + 1) + RB * RB),
        invd(2 * RB * (RB + 1) + 2 * RB * RB), X(2 * RB * (RB + 1) + 2 * RB * RB + RB + (RB & 1)),
        scr(X + kSolveRows * (RB + 1)), red(scr + 8 * 64), lam(red + 32), total(lam + RB) {}
};

template <int RB, bool LAST>
__global__ void __launch_bounds__(kSolveRows, 2) upd_solve_kernel(UpdArgs a, int n, int nch) {
  extern __shared__ __align__(16) double sm[];
  constexpr SolveSmem L(RB);
  double* U = sm + L.U;         // U pre-shifted (or pinv), pitch RP
  double* V = sm + L.V;         // U^T pre-shifted, pitch RP
  double* Hs = sm + L.H;        // last mode: Hadamard of G_0 .. G_{N-2} (R x R)
  double* Gs = sm + L.G;        // the refreshed Gramian (R x R)
  double* invd = sm + L.invd;   // 1 / U[a][a]
  double* X = sm + L.X;         // kSolveRows x P: M rows, then the solved rows
  double* scr = sm + L.scr;
  double* red = sm + L.red;
  double* lam = sm + L.lam;     // (cold path)
  __shared__ int s_last;
  const int tid = threadIdx.x;
#ifdef CALS_SOLVE_PROFILE
  const long long t_entry = clock64();
#endif
  const int sb = blockIdx.x / nch;
  const int chunk = blockIdx.x - sb * nch;
  const int na = *a.n_active;
  if (sb >= na) return;
  // CTA order: with rev, the last registry slot first.  The block scheduler
  // gives the first ~148 CTAs an SM of their own and doubles up the rest;
  // queues built in rank order (build_models) put the widest models last,
  // and their chains are the kernel's critical path.  Results do not depend
  // on which CTA solves a model.
  const int slot = a.rev ? na - 1 - sb : sb;
  const int4 si = a.slot_info[slot];
  const int k = si.x, R = si.y, off = si.z;
  const long long go = si.w;
  const int pf = a.pflag[k];
  const long long ld = a.ld;
  const int rows = (int)param_at(a.dims, n);
  double* const Fn = param_at(a.F, n);
  const int r0 = chunk * kSolveRows;
  const int cnt = min(kSolveRows, rows - r0);
  const int P = fast_pitch(R);
  const int RP = R + (R & 1);
#ifdef CALS_SOLVE_PROFILE
  if (tid == 0 && blockIdx.x < 2048) g_solve_prof[n][blockIdx.x][0] = R;
#endif
  SOLVE_STAMP(1)
  if (pf == kPrepFailed) {  // failed earlier in this iteration (driver.py:218-219)
    if (LAST && chunk == 0 && tid == 0) finish_model(a, k, 0.0, 0.0, false);
    if (a.lo[0].src == n || a.lo[1].src == n) {  // the factor stays: its slices still feed
      griddep_wait();                                 // the later contraction
      slice_lo_targets(a, n, off, R, Fn + off, a.ld);
    }
    return;
  }
  DecideIn din{};
  int ls_on = 0;
  if (LAST && tid == 0) {  // independent loads, consumed at the very end
    EngState* st = a.st;
    din.it = st->iters[k] + 1;
    din.failed = st->failed[k];
    din.f_prev = st->f_prev[k];
    din.tol = st->tol;
    din.sqnorm = st->sqnorm;
    din.max_iterations = st->max_iterations;
    ls_on = st->ls_enabled;
  }
  // U, U^T (or pinv) and, for the last mode, H: written by prep (before)
  {
    const double* src = a.ubuf + 3 * go;
    if (pf == kPrepChol) {
      // pre-shifted rows for the rotation solve (solve_row_exact)
      for (int idx = tid; idx < R * RP; idx += kSolveRows) {
        const int r = idx / RP, j = idx - r * RP;
        const int cu = r + 1 + j, cv = r - 1 - j;
        U[idx] = cu < R ? src[r * R + cu] : 0.0;
        V[idx] = cv >= 0 ? src[R * R + r * R + cv] : 0.0;
      }
      for (int r = tid; r < R; r += kSolveRows) invd[r] = src[r * R + r];
    } else {
      for (int idx = tid; idx < R * R; idx += kSolveRows) U[idx] = src[idx];  // pinv, pitch R
    }
    if (LAST)
      for (int idx = tid; idx < R * R; idx += kSolveRows) Hs[idx] = src[2 * R * R + idx];
  }
  // The reference checks the whole M block before touching the factor
  // (als.py:84-85): every chunk scans all of it (one chunk at <= 256 rows),
  // staging its own rows on the way, so all chunks reach the same verdict.
  // M_n straight from the contraction's split-K partials (non-last modes,
  // SplitDefer): summed here in split order instead of by split_reduce_kernel
  const bool parts = !LAST && a.mS > 1;
  const double* Mb = (parts ? a.mpart : a.Mout) + off;
  const long long ldm = parts ? a.mpart_ld : ld;
  int bad = pf == kPrepBadH;
  // everything above came from earlier kernels (plan, prep); M_n is the
  // output of the grid right before this one (programmatic launch)
  griddep_wait();
  SOLVE_STAMP(8)
  // element e = i * R + c of the block walked with stride kSolveRows without
  // integer divisions: (i, c) advance by (dq, dr) per step
  const int dq = kSolveRows / R, dr = kSolveRows - dq * R;
  if (parts) {
    // B elements per round with up to G partial blocks of each in flight at
    // once: a c3 block (S = 11) costs one L2 round trip per round instead of
    // one per group of four partials
    constexpr int B = 4, G = 10;
    const int S = a.mS;
    const long long ps = a.mpart_stride;
    int i = tid / R, c = tid - (tid / R) * R;
    while (i < rows) {
      int eo[B], xi[B];
      double v[B];
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const bool ok = i < rows;
        const int il = i - r0;
        eo[u] = ok ? int((long long)i * ldm + c) : -1;
        xi[u] = ok && il >= 0 && il < cnt ? il * P + c : -1;
        v[u] = ok ? Mb[eo[u]] : 0.0;
        i += dq;
        c += dr;
        if (c >= R) {
          c -= R;
          ++i;
        }
      }
      // partials 1 .. S-1 added in order (split_reduce_kernel's); a lane
      // past S adds nothing (not even +0.0, which would turn -0.0 into +0.0)
      for (int s = 1; s < S; s += G) {
        double w[G][B];
#pragma unroll
        for (int t = 0; t < G; ++t)
#pragma unroll
          for (int u = 0; u < B; ++u)
            w[t][u] = (s + t < S && eo[u] >= 0) ? Mb[(s + t) * ps + eo[u]] : 0.0;
#pragma unroll
        for (int t = 0; t < G; ++t)
#pragma unroll
          for (int u = 0; u < B; ++u)
            if (s + t < S) v[u] += w[t][u];
      }
#pragma unroll
      for (int u = 0; u < B; ++u) {
        bad |= !isfinite(v[u]);
        if (xi[u] >= 0) X[xi[u]] = v[u];
      }
    }
  } else {
    int i = tid / R, c = tid - (tid / R) * R;
    while (i < rows) {
      double v[16];
      int iu[16], cu[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        iu[u] = i;
        cu[u] = c;
        v[u] = i < rows ? Mb[(long long)i * ld + c] : 0.0;
        i += dq;
        c += dr;
        if (c >= R) {
          c -= R;
          ++i;
        }
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        bad |= !isfinite(v[u]);
        const int il = iu[u] - r0;
        if (iu[u] < rows && il >= 0 && il < cnt) X[il * P + cu[u]] = v[u];
      }
    }
  }
  const int any_bad = __syncthreads_or(bad);
  SOLVE_STAMP(2)
  if (any_bad) {
    if (chunk == 0 && tid == 0) {
      a.failed[k] = 1;
      if (LAST) finish_model(a, k, 0.0, 0.0, false);
    }
    slice_lo_targets(a, n, off, R, Fn + off, a.ld);
    return;
  }
  int sbad = 0;
  SOLVE_STAMP(3)
  if (tid < cnt) {
    double* x = X + tid * P;
    if (pf == kPrepChol) {
      solve_row_dispatch<RB>(R, x, U, V, invd);
      for (int c = 0; c < R; ++c) sbad |= !isfinite(x[c]);
    } else {
      apply_pinv_row<RB>(x, U, R);
    }
  }
  __syncthreads();
  SOLVE_STAMP(4)
  // coalesced store of the solved rows (+ the last mode's <A, M> partial)
  double dot = 0.0;
  {
    double* Ac = Fn + (long long)r0 * ld + off;
    const double* Mc = Mb + (long long)r0 * ld;
    int i = tid / R, c = tid - (tid / R) * R;
#pragma unroll 16
    for (; i < cnt;) {
      const double v = X[i * P + c];
      Ac[(long long)i * ld + c] = v;
      if (LAST) dot = fma(v, Mc[(long long)i * ld + c], dot);
      i += dq;
      c += dr;
      if (c >= R) {
        c -= R;
        ++i;
      }
    }
  }
  SOLVE_STAMP(9)
  // Gramian refresh from the solved rows (driver.py:234)
  tile_gram_tc(X, P, cnt, R, scr, Gs);
  double inner = 0.0;
  if (LAST) {
    inner = block_sum(dot, red);  // (its barriers also publish Gs)
    if (nch > 1 && tid == 0) a.ipart[(long long)k * nch + chunk] = inner;
  }
  sbad = __syncthreads_or(sbad);
  SOLVE_STAMP(5)
  double* Gn = a.grams + (long long)n * a.gram_stride + go;
  bool redo = sbad != 0;
  if (nch > 1) {
    // this chunk's (upper) partial, then arrival: the last chunk finishes
    double* gp = a.gpart + go * nch + (long long)chunk * R * R;
    for (int idx = tid; idx < R * R; idx += kSolveRows) gp[idx] = Gs[idx];
    if (sbad && tid == 0) a.solbad[k] = 1;
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(&a.arrive[k], 1) == nch - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    redo = *(volatile int*)&a.solbad[k] != 0;
    __syncthreads();
    if (tid == 0) {
      a.arrive[k] = 0;
      a.solbad[k] = 0;
    }
    if (!redo) {
      for (int idx = tid; idx < R * R; idx += kSolveRows) {
        double s = 0.0;
        for (int ch = 0; ch < nch; ++ch) s += a.gpart[go * nch + (long long)ch * R * R + idx];
        Gs[idx] = s;
      }
      if (LAST) {
        inner = 0.0;
        for (int ch = 0; ch < nch; ++ch) inner += a.ipart[(long long)k * nch + ch];
      }
    }
  }
  double* Afull = Fn + off;
  if (redo) {
    // cho_solve gave a non-finite entry: the whole block again with pinv(H)
    // (als.py:88-96); H from the unchanged Gramians of the other modes
    hadamard_others(a.grams, a.gram_stride, go, a.order, n, R, U, tid, kSolveRows);
    __syncthreads();
    block_pinv(U, X, lam, R);
    for (long long e = tid; e < (long long)rows * R; e += kSolveRows) {
      const int i = int(e / R), c = int(e % R);
      const double* m = Mb + (long long)i * ldm;
      double s = 0.0;
      for (int b = 0; b < R; ++b) {
        double mb = m[b];
        if (parts)
          for (int q = 1; q < a.mS; ++q) mb += m[q * a.mpart_stride + b];
        s = fma(mb, U[b * R + c], s);
      }
      Afull[(long long)i * ld + c] = s;
    }
    __syncthreads();
    for (int idx = tid; idx < R * R; idx += kSolveRows) {
      const int r = idx / R, c = idx - r * R;
      const int lo = r <= c ? r : c, hi = r <= c ? c : r;
      double s = 0.0;
      for (int i = 0; i < rows; ++i)
        s = fma(Afull[(long long)i * ld + lo], Afull[(long long)i * ld + hi], s);
      Gs[idx] = s;
    }
    if (LAST) {
      double part = 0.0;
      for (long long e = tid; e < (long long)rows * R; e += kSolveRows) {
        const long long i = e / R;
        const int c = int(e - i * R);
        part = fma(Afull[i * ld + c], Mb[i * ld + c], part);
      }
      inner = block_sum(part, red);
    }
  }
  __syncthreads();  // Gs final
  for (int idx = tid; idx < R * R; idx += kSolveRows) Gn[idx] = Gs[idx];
  SOLVE_STAMP(6)
  // nch == 1 for a fusion source (setup_lo_fusion): X holds every solved row
  // unless the pinv redo used it as scratch
  if (redo)
    slice_lo_targets(a, n, off, R, Fn + off, a.ld);
  else
    slice_lo_targets(a, n, off, R, X, P);
  SOLVE_STAMP(10)
  if (!LAST) return;
  // fast error (als.py:99-115): sum of the Hadamard of all Gramians, folded
  // ascending -- (G_0 o .. o G_{N-2}) from prep, then o G_{N-1}
  double mpart = 0.0;
  for (int idx = tid; idx < R * R; idx += kSolveRows) mpart += Hs[idx] * Gs[idx];
  const double msq = block_sum(mpart, red);
  SOLVE_STAMP(11)
  if (tid == 0) finish_model_pre(a, k, msq, inner, din, ls_on);
  SOLVE_STAMP(7)
}

#ifdef CALS_SOLVE_PROFILE
int debug_solve_prof(long long* host, size_t bytes) {
  return cudaMemcpyFromSymbol(host, g_solve_prof, bytes < sizeof(g_solve_prof) ? bytes
                                                                               : sizeof(g_solve_prof))
             == cudaSuccess ? 0 : -1;
}
#endif

void split_kernels_for(int rb, PrepKernel* prep, SolveKernel* solve, SolveKernel* last,
                       size_t* smem) {
  switch (rb) {
    case 8: *prep = upd_prep_kernel<8>; *solve = upd_solve_kernel<8, false>;
            *last = upd_solve_kernel<8, true>; break;
    case 16: *prep = upd_prep_kernel<16>; *solve = upd_solve_kernel<16, false>;
             *last = upd_solve_kernel<16, true>; break;
    case 24: *prep = upd_prep_kernel<24>; *solve = upd_solve_kernel<24, false>;
             *last = upd_solve_kernel<24, true>; break;
    default: *prep = upd_prep_kernel<32>; *solve = upd_solve_kernel<32, false>;
             *last = upd_solve_kernel<32, true>; break;
  }
  *smem = solve_smem_bytes(rb);
}

}  // namespace cals
