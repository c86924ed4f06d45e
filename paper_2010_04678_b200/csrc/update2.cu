// Split per-model update kernels (see update2.cuh for the design).
#include "update.cuh"
#include "update2.cuh"

namespace cals {

// G = A^T A of the column block A[i][r] (rows x R, row stride ld) by one warp:
// the block goes through shared memory 32 rows at a time (pitch P odd), each
// lane accumulates its (a, b) pairs over ascending rows (the same chain per
// pair as block_gram_fast), upper triangle mirrored.
template <int RB>
__device__ __forceinline__ void warp_gram(const double* __restrict__ A, long long ld, int rows,
                                          int R, double* __restrict__ T, double* __restrict__ G) {
  constexpr int NP = (RB * (RB + 1) / 2 + 31) / 32;
  const int lane = threadIdx.x & 31;
  const int P = fast_pitch(R);
  const int npairs = R * (R + 1) / 2;
  int pa[NP], pb[NP];
  double acc[NP];
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    const int p = lane + 32 * j;
    acc[j] = 0.0;
    pa[j] = -1;
    pb[j] = 0;
    if (p < npairs) {
      int aa = 0, rem = p;
      while (rem >= R - aa) {
        rem -= R - aa;
        ++aa;
      }
      pa[j] = aa;
      pb[j] = aa + rem;
    }
  }
  for (int base = 0; base < rows; base += 32) {
    const int cnt = min(32, rows - base);
    stage_block(A + (long long)base * ld, ld, cnt, R, P, T, lane, 32);
    __syncwarp();
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      if (pa[j] < 0) continue;
      const double* xa = T + pa[j];
      const double* xb = T + pb[j];
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
    __syncwarp();
  }
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    if (pa[j] < 0) continue;
    G[pa[j] * R + pb[j]] = acc[j];
    G[pb[j] * R + pa[j]] = acc[j];
  }
}

// H = Hadamard of the Gramians of every mode but n (ascending), R x R, into
// shared memory; returns (to every thread of the calling group) whether any
// entry is non-finite.
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
  if (n == 0) {
    if (a.fresh[k]) {  // Gramians of the admitted starting point (driver.py:203-205)
      for (int i = 1; i < N; ++i)
        warp_gram<RB>(a.F[i] + off, a.ld, (int)a.dims[i], R, T, a.grams + i * gs + go);
      if (lane == 0) a.fresh[k] = 0;
    }
  } else {  // the factor updated last (driver.py:234)
    warp_gram<RB>(a.F[n - 1] + off, a.ld, (int)a.dims[n - 1], R, T,
                  a.grams + (n - 1) * gs + go);
  }
  __syncwarp();
  const int bad = __any_sync(0xffffffffu, hadamard_others(a.grams, gs, go, N, n, R, H, lane, 32));
  if (bad) {  // non-finite h: update_factor raises (als.py:84-85)
    if (lane == 0) a.pflag[k] = kPrepBadH;
    return;
  }
  __syncwarp();
  warp_cholesky_rb<RB>(H, R, invd, &flag);
  __syncwarp();
  double* U = a.ubuf + go;
  if (flag) {
    for (int idx = lane; idx < R * R; idx += 32) {
      const int r = idx / R, c = idx - r * R;
      U[idx] = r < c ? H[idx] : (r == c ? invd[r] : 0.0);
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

// x <- m P for one row (als.py:96: m @ pinv), b ascending as block_apply_pinv
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

template <int RB, bool LAST>
__global__ void __launch_bounds__(kSolveRows, 3) upd_solve_kernel(UpdArgs a, int n, int nch) {
  extern __shared__ __align__(16) double sm[];
  double* U = sm;                  // RB * RB
  double* invd = U + RB * RB;      // RB
  double* X = invd + RB;           // kSolveRows * P
  double* red = X + kSolveRows * (RB + 1);  // 32
  double* lam = red + 32;          // RB (cold path)
  __shared__ int s_last;
  const int tid = threadIdx.x;
  const int slot = blockIdx.x / nch;
  const int chunk = blockIdx.x - slot * nch;
  const int na = *a.n_active;
  const int4 si = a.slot_info[slot];
  if (slot >= na) return;
  const int k = si.x, R = si.y, off = si.z;
  const long long go = si.w;
  const int pf = a.pflag[k];
  const long long ld = a.ld;
  const int rows = (int)a.dims[n];
  const int r0 = chunk * kSolveRows;
  const int cnt = min(kSolveRows, rows - r0);
  const int P = fast_pitch(R);
  if (pf == kPrepFailed) {  // failed earlier in this iteration (driver.py:218-219)
    if (LAST && chunk == 0 && tid == 0) finish_model(a, k, 0.0, 0.0, false);
    return;
  }
  for (int idx = tid; idx < R * R; idx += kSolveRows) {
    const double u = a.ubuf[go + idx];
    U[idx] = u;
    if (pf == kPrepChol && idx / R == idx % R) invd[idx / R] = u;
  }
  // The reference checks the whole M block before touching the factor
  // (als.py:84-85): every chunk scans all of it (L2-resident, just written),
  // staging its own rows on the way, so all chunks reach the same verdict.
  const double* Mb = a.Mout + off;
  int bad = pf == kPrepBadH;
  {
    const int total = rows * R;
    for (int e0 = tid; e0 < total; e0 += 4 * kSolveRows) {
      double v[4];
      int ii[4], cc[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + u * kSolveRows;
        ii[u] = e / R;
        cc[u] = e - ii[u] * R;
        v[u] = e < total ? Mb[(long long)ii[u] * ld + cc[u]] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        bad |= !isfinite(v[u]);
        const int i = ii[u] - r0;
        if (e0 + u * kSolveRows < total && i >= 0 && i < cnt) X[i * P + cc[u]] = v[u];
      }
    }
  }
  if (__syncthreads_or(bad)) {
    if (chunk == 0 && tid == 0) {
      a.failed[k] = 1;
      if (LAST) finish_model(a, k, 0.0, 0.0, false);
    }
    return;
  }
  int sbad = 0;
  if (tid < cnt) {
    double* x = X + tid * P;
    if (pf == kPrepChol) {
      if (RB <= 8 || R <= 8)
        solve_row_reg<(RB < 8 ? RB : 8)>(x, U, invd, R);
      else if (RB <= 16 || R <= 16)
        solve_row_reg<(RB < 16 ? RB : 16)>(x, U, invd, R);
      else if (RB <= 24 || R <= 24)
        solve_row_reg<(RB < 24 ? RB : 24)>(x, U, invd, R);
      else
        solve_row_reg<RB>(x, U, invd, R);
      for (int c = 0; c < R; ++c) sbad |= !isfinite(x[c]);
    } else {
      apply_pinv_row<RB>(x, U, R);
    }
  }
  __syncthreads();
  double dot = 0.0;
  {
    double* Ac = a.F[n] + (long long)r0 * ld + off;
    const double* Mc = Mb + (long long)r0 * ld;
    const int total = cnt * R;
    for (int e = tid; e < total; e += kSolveRows) {
      const int i = e / R, c = e - i * R;
      const double v = X[i * P + c];
      Ac[(long long)i * ld + c] = v;
      if (LAST) dot = fma(v, Mc[(long long)i * ld + c], dot);
    }
  }
  if (LAST) {
    // partial Gramian (upper triangle, ascending rows of this chunk) and
    // partial inner product of the chunk
    constexpr int NPB = (RB * (RB + 1) / 2 + kSolveRows - 1) / kSolveRows;
    const int npairs = R * (R + 1) / 2;
    double* gp = a.gpart + go * nch + (long long)chunk * R * R;
#pragma unroll
    for (int j = 0; j < NPB; ++j) {
      const int p = tid + j * kSolveRows;
      if (p < npairs) {
        int aa = 0, rem = p;
        while (rem >= R - aa) {
          rem -= R - aa;
          ++aa;
        }
        const int bb = aa + rem;
        const double* xa = X + aa;
        const double* xb = X + bb;
        double s = 0.0;
        int r = 0;
        for (; r + 4 <= cnt; r += 4) {
          s = fma(xa[r * P], xb[r * P], s);
          s = fma(xa[(r + 1) * P], xb[(r + 1) * P], s);
          s = fma(xa[(r + 2) * P], xb[(r + 2) * P], s);
          s = fma(xa[(r + 3) * P], xb[(r + 3) * P], s);
        }
        for (; r < cnt; ++r) s = fma(xa[r * P], xb[r * P], s);
        gp[aa * R + bb] = s;
      }
    }
    const double inner = block_sum(dot, red);
    if (tid == 0) a.ipart[(long long)k * nch + chunk] = inner;
  }
  if (__syncthreads_or(sbad) && tid == 0) a.solbad[k] = 1;
  // arrival: the last chunk of the model finishes it
  __threadfence();
  if (tid == 0) s_last = atomicAdd(&a.arrive[k], 1) == nch - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const bool redo = *(volatile int*)&a.solbad[k] != 0;
  __syncthreads();
  if (tid == 0) {
    a.arrive[k] = 0;
    a.solbad[k] = 0;
  }
  const double* Mfull = Mb;
  double* Afull = a.F[n] + off;
  if (redo) {
    // cho_solve gave a non-finite entry: the whole block again with pinv(H)
    // (als.py:88-96); H from the unchanged Gramians of the other modes
    hadamard_others(a.grams, a.gram_stride, go, a.order, n, R, U, tid, kSolveRows);
    __syncthreads();
    block_pinv(U, X, lam, R);
    for (long long e = tid; e < (long long)rows * R; e += kSolveRows) {
      const int i = int(e / R), c = int(e % R);
      const double* m = Mfull + (long long)i * ld;
      double s = 0.0;
      for (int b = 0; b < R; ++b) s = fma(m[b], U[b * R + c], s);
      Afull[(long long)i * ld + c] = s;
    }
    __syncthreads();
  }
  if (!LAST) return;
  // Gramian of the last mode and the fast error (als.py:99-115)
  double* G = a.grams + (long long)(a.order - 1) * a.gram_stride + go;
  double inner = 0.0;
  if (!redo) {
    for (int idx = tid; idx < R * R; idx += kSolveRows) {
      const int r = idx / R, c = idx - r * R;
      const int u = r <= c ? idx : c * R + r;
      double s = 0.0;
      for (int ch = 0; ch < nch; ++ch) s += a.gpart[go * nch + (long long)ch * R * R + u];
      G[idx] = s;
    }
    for (int ch = 0; ch < nch; ++ch) inner += a.ipart[(long long)k * nch + ch];
  } else {
    for (int idx = tid; idx < R * R; idx += kSolveRows) {
      const int r = idx / R, c = idx - r * R;
      const int lo = r <= c ? r : c, hi = r <= c ? c : r;
      double s = 0.0;
      for (int i = 0; i < rows; ++i)
        s = fma(Afull[(long long)i * ld + lo], Afull[(long long)i * ld + hi], s);
      G[idx] = s;
    }
    double part = 0.0;
    for (long long e = tid; e < (long long)rows * R; e += kSolveRows) {
      const long long i = e / R;
      const int c = int(e - i * R);
      part = fma(Afull[i * ld + c], Mfull[i * ld + c], part);
    }
    inner = block_sum(part, red);
  }
  __syncthreads();
  double mpart = 0.0;
  for (int idx = tid; idx < R * R; idx += kSolveRows) {
    double h = a.grams[go + idx];
    for (int i = 1; i < a.order; ++i) h *= a.grams[i * a.gram_stride + go + idx];
    mpart += h;
  }
  const double msq = block_sum(mpart, red);
  if (tid == 0) finish_model(a, k, msq, inner, true);
}

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
