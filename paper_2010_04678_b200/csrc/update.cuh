// Per-model ALS factor update on the block-diagonal structure of the fused
// problem: Hadamard of the other modes' Gramians, upper Cholesky of the
// R x R normal matrix, row-wise triangular solves, eigen-pinv fallback,
// Gram refresh and the fast error / fit.  One thread block owns one model.
//
// Reference semantics restated (pkg/src/cals):
//   hadamard_fold ascending, excluding mode n ......... driver.py:223-225, tensor.py:169-180
//   update_factor: cho_factor(upper)+cho_solve, on
//     LinAlgError / non-finite -> eigh pinv, cutoff
//     1e-12 * max(lambda_max, 0); ValueError on
//     non-finite input .................................. als.py:74-96
//   gramian: upper triangle computed, lower mirrored .. tensor.py:183-188
//   fast_error with the e > 0 ? e : 0 clamp ............ als.py:99-115
//   fit = 1 - sqrt(e)/sqrt(||T||^2) ................... als.py:118-124
#pragma once

#include "common.cuh"

namespace cals {

constexpr int kUpdThreads = 256;
// Generic update path limits: the R x R matrix of the block routines below
// lives in shared memory up to kSmemRankMax, in global scratch above it;
// the row tile (R x >= 32 threads' rows) bounds the rank at kMaxRank.
constexpr int kSmemRankMax = 128;
constexpr int kMaxRank = 512;
// per-block global scratch of the engine's update kernel (doubles): V, Hsave
// (R^2 each), lam (R), and H (R^2) above kSmemRankMax
__host__ __device__ constexpr long long upd_scratch_doubles(int R) {
  return 2LL * R * R + R + (R > kSmemRankMax ? (long long)R * R : 0LL);
}

// Deterministic block sum (blockDim.x a multiple of 32; `red` has >= 32
// doubles): an xor butterfly inside each warp (partners add the same two
// values, so every lane holds the same bits), then the warp sums in warp
// order.  Two barriers instead of a log2(blockDim) smem tree.
__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = red[0];
  for (int i = 1; i < nw; ++i) s += red[i];
  __syncthreads();  // red reusable
  return s;
}

// G = A^T A of the column block A[i][off + r] (rows x R, row stride ld):
// upper triangle summed over ascending rows, then mirrored.
__device__ inline void block_gram(const double* F, long long ld, int off, int rows, int R,
                                  double* G) {
  const int pairs = R * (R + 1) / 2;
  for (int idx = threadIdx.x; idx < pairs; idx += blockDim.x) {
    // decode idx -> (a, b), a <= b, row-major over the upper triangle
    int a = 0, rem = idx;
    while (rem >= R - a) {
      rem -= R - a;
      ++a;
    }
    const int b = a + rem;
    const double* pa = F + off + a;
    const double* pb = F + off + b;
    double s = 0.0;
    for (int i = 0; i < rows; ++i) s = fma(pa[(long long)i * ld], pb[(long long)i * ld], s);
    G[a * R + b] = s;
    G[b * R + a] = s;
  }
}

// In-place upper Cholesky of the R x R matrix in shared memory (upper
// triangle read and overwritten with U, H = U^T U).  Warp 0 factors; the
// result flag is returned to every thread.  Fails like dpotrf: pivot <= 0
// or NaN.
__device__ inline bool block_cholesky_upper(double* H, int R, int* flag) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    bool ok = true;
    for (int j = 0; j < R && ok; ++j) {
      const double d = H[j * R + j];
      ok = d > 0.0;  // false for NaN
      if (!ok) break;
      const double u = sqrt(d);
      __syncwarp();
      if (lane == 0) H[j * R + j] = u;
      for (int b = j + 1 + lane; b < R; b += 32) H[j * R + b] /= u;
      __syncwarp();
      for (int b = j + 1 + lane; b < R; b += 32) {
        const double ujb = H[j * R + b];
        for (int a = j + 1; a <= b; ++a) H[a * R + b] = fma(-H[j * R + a], ujb, H[a * R + b]);
      }
      __syncwarp();
    }
    if (lane == 0) *flag = ok ? 1 : 0;
  }
  __syncthreads();
  return *flag != 0;
}

// Rows x = U^{-1} U^{-T} m for every row of the M block (dpotrs order:
// forward with U^T, back with U).  X is shared scratch [R][nthr].  Writes the
// solution into A; returns (block-wide) whether every entry is finite.
__device__ inline bool block_row_solve(const double* U, int R, const double* Mb, long long ldm,
                                       int rows, double* A, long long lda, double* X, int nthr) {
  int bad = 0;
  const int t = threadIdx.x;
  if (t < nthr) {
    for (int i = t; i < rows; i += nthr) {
      const double* m = Mb + (long long)i * ldm;
      for (int a = 0; a < R; ++a) X[a * nthr + t] = m[a];
      for (int a = 0; a < R; ++a) {
        double s = X[a * nthr + t];
        for (int k = 0; k < a; ++k) s = fma(-U[k * R + a], X[k * nthr + t], s);
        X[a * nthr + t] = s / U[a * R + a];
      }
      for (int a = R - 1; a >= 0; --a) {
        double s = X[a * nthr + t];
        for (int k = a + 1; k < R; ++k) s = fma(-U[a * R + k], X[k * nthr + t], s);
        X[a * nthr + t] = s / U[a * R + a];
      }
      double* o = A + (long long)i * lda;
      for (int a = 0; a < R; ++a) {
        const double v = X[a * nthr + t];
        bad |= !isfinite(v);
        o[a] = v;
      }
    }
  }
  return __syncthreads_or(bad) == 0;
}

// Cyclic Jacobi eigen-decomposition of the symmetric R x R matrix H (full
// storage), eigenvectors into V (columns).  Warp 0 only; cold path.
__device__ inline void warp_jacobi(double* H, double* V, int R) {
  const int lane = threadIdx.x & 31;
  for (int idx = lane; idx < R * R; idx += 32) V[idx] = (idx / R == idx % R) ? 1.0 : 0.0;
  __syncwarp();
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int idx = lane; idx < R * R; idx += 32) {
      const double v = H[idx] * H[idx];
      tot += v;
      if (idx / R != idx % R) off += v;
    }
    for (int o = 16; o > 0; o >>= 1) {
      off += __shfl_xor_sync(0xffffffffu, off, o);
      tot += __shfl_xor_sync(0xffffffffu, tot, o);
    }
    if (off <= 1e-32 * tot || off == 0.0) break;
    for (int p = 0; p < R - 1; ++p)
      for (int q = p + 1; q < R; ++q) {
        const double apq = H[p * R + q];
        if (apq == 0.0) continue;
        const double app = H[p * R + p], aqq = H[q * R + q];
        const double theta = (aqq - app) / (2.0 * apq);
        const double tt =
            (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(tt * tt + 1.0), s = tt * c;
        __syncwarp();
        for (int k = lane; k < R; k += 32) {  // columns p, q
          const double hkp = H[k * R + p], hkq = H[k * R + q];
          H[k * R + p] = c * hkp - s * hkq;
          H[k * R + q] = s * hkp + c * hkq;
          const double vkp = V[k * R + p], vkq = V[k * R + q];
          V[k * R + p] = c * vkp - s * vkq;
          V[k * R + q] = s * vkp + c * vkq;
        }
        __syncwarp();
        for (int k = lane; k < R; k += 32) {  // rows p, q
          const double hpk = H[p * R + k], hqk = H[q * R + k];
          H[p * R + k] = c * hpk - s * hqk;
          H[q * R + k] = s * hpk + c * hqk;
        }
        __syncwarp();
      }
  }
}

// Pseudo-inverse fallback: H (smem, full symmetric, destroyed) -> P = pinv(H)
// written into H; V and lam are scratch (R*R and R doubles).
__device__ inline void block_pinv(double* H, double* V, double* lam, int R) {
  if (threadIdx.x < 32) {
    warp_jacobi(H, V, R);
    __syncwarp();
    if (threadIdx.x == 0) {
      double lmax = -INFINITY;
      for (int k = 0; k < R; ++k) {
        lam[k] = H[k * R + k];
        lmax = fmax(lmax, lam[k]);
      }
      const double cut = 1e-12 * fmax(lmax, 0.0);
      for (int k = 0; k < R; ++k) lam[k] = lam[k] > cut ? 1.0 / lam[k] : 0.0;
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < R * R; idx += blockDim.x) {
    const int a = idx / R, b = idx % R;
    double s = 0.0;
    for (int k = 0; k < R; ++k) s = fma(V[a * R + k] * lam[k], V[b * R + k], s);
    H[idx] = s;
  }
  __syncthreads();
}

// rows of A = m @ P
__device__ inline void block_apply_pinv(const double* P, int R, const double* Mb, long long ldm,
                                        int rows, double* A, long long lda) {
  for (long long e = threadIdx.x; e < (long long)rows * R; e += blockDim.x) {
    const int i = int(e / R), a = int(e % R);
    const double* m = Mb + (long long)i * ldm;
    double s = 0.0;
    for (int b = 0; b < R; ++b) s = fma(m[b], P[b * R + a], s);
    A[(long long)i * lda + a] = s;
  }
  __syncthreads();
}

// Full update of one column block: returns false if the inputs were
// non-finite (the reference raises ValueError -> instance FAILED).
// H (smem R*R) must hold the Hadamard product on entry; Hsave (R*R, any
// memory) receives a copy for the pinv path; X/V/lam are scratch.
__device__ inline bool block_update(double* H, double* Hsave, double* V, double* lam, double* X,
                                    int nthr, int R, const double* Mb, long long ldm, int rows,
                                    double* A, long long lda, int* flag) {
  int bad = 0;
  for (int idx = threadIdx.x; idx < R * R; idx += blockDim.x) {
    bad |= !isfinite(H[idx]);
    Hsave[idx] = H[idx];
  }
  for (long long e = threadIdx.x; e < (long long)rows * R; e += blockDim.x)
    bad |= !isfinite(Mb[(e / R) * ldm + e % R]);
  if (__syncthreads_or(bad)) return false;
  bool ok = block_cholesky_upper(H, R, flag);
  if (ok) ok = block_row_solve(H, R, Mb, ldm, rows, A, lda, X, nthr);
  if (!ok) {
    for (int idx = threadIdx.x; idx < R * R; idx += blockDim.x) H[idx] = Hsave[idx];
    __syncthreads();
    block_pinv(H, V, lam, R);
    block_apply_pinv(H, R, Mb, ldm, rows, A, lda);
  }
  return true;
}

// ---------------------------------------------------------------------------
// Fast path for R <= 32 (every config rank): compact loops only -- the
// update runs once per model per mode, so straight-line unrolled code would
// be bound by instruction fetch.  One thread per factor row solves in place
// in a shared-memory chunk Xs (row pitch P odd -> conflict-free), in
// dpotrs/dtrsm order (forward: for each a subtract k ascending; back: k
// descending) multiplying by the reciprocal diagonal as OpenBLAS's packed
// trsm kernels do; the same chunk feeds the Gram refresh (pair sums over
// rows in ascending order -> deterministic).

constexpr int kFastR = 32;
constexpr int kFastNP = (kFastR * (kFastR + 1) / 2 + kUpdThreads - 1) / kUpdThreads;

__device__ __forceinline__ int fast_pitch(int R) { return (R & 1) ? R : R + 1; }

// pairs per thread for rank bucket RB
__host__ __device__ constexpr int fast_np(int RB) { return (RB * (RB + 1) / 2 + kUpdThreads - 1) / kUpdThreads; }
template <int NP>
struct FastPairsT {
  int a[NP], b[NP];
  double acc[NP];
  __device__ void init(int R) {
    const int npairs = R * (R + 1) / 2;
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      const int p = threadIdx.x + j * kUpdThreads;
      acc[j] = 0.0;
      a[j] = -1;
      b[j] = -1;
      if (p < npairs) {
        int aa = 0, rem = p;
        while (rem >= R - aa) {
          rem -= R - aa;
          ++aa;
        }
        a[j] = aa;
        b[j] = aa + rem;
      }
    }
  }
  __device__ void accumulate(const double* Xs, int P, int cnt) {
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      if (a[j] < 0) continue;
      const double* pa = Xs + a[j];
      const double* pb = Xs + b[j];
      double s = acc[j];
      int r = 0;
      for (; r + 4 <= cnt; r += 4) {
        const double x0 = pa[r * P], y0 = pb[r * P], x1 = pa[(r + 1) * P], y1 = pb[(r + 1) * P];
        const double x2 = pa[(r + 2) * P], y2 = pb[(r + 2) * P], x3 = pa[(r + 3) * P],
                     y3 = pb[(r + 3) * P];
        s = fma(x0, y0, s);
        s = fma(x1, y1, s);
        s = fma(x2, y2, s);
        s = fma(x3, y3, s);
      }
      for (; r < cnt; ++r) s = fma(pa[r * P], pb[r * P], s);
      acc[j] = s;
    }
  }
  __device__ void store(double* G, int R) const {
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      if (a[j] < 0) continue;
      G[a[j] * R + b[j]] = acc[j];
      G[b[j] * R + a[j]] = acc[j];
    }
  }
};

// Upper Cholesky of H (smem, R <= 32) by warp 0 with the matrix in
// registers: lane b holds column b, rotated by one row per step so the
// current pivot row is always col[0] (static register indices, compact
// loop).  Step k: pivot from lane k, u = sqrt, inv = 1/u (uniform), row k
// of U = H[k][b] * inv (dpotf2: DSCAL by 1/ajj), trailing update
// H[a][b] -= U[k][a] U[k][b] with U[k][a] broadcast by shuffles.  U is
// written back over the upper triangle; inv_diag[k] = 1/U[k][k].  Fails like
// dpotrf (pivot <= 0 or NaN).
template <int RB>
__device__ __forceinline__ void warp_cholesky_rb(double* __restrict__ H, int R,
                                                 double* __restrict__ inv_diag, int* flag) {
  const int lane = threadIdx.x;
  double col[RB];  // lane b: column b, rows k.. (rotated: col[0] is the pivot row)
#pragma unroll
  for (int a = 0; a < RB; ++a) col[a] = (a < R && lane < R && a <= lane) ? H[a * R + lane] : 0.0;
  bool ok = true;
  // The k loop stays rolled: one compact body (RB - 1 shuffles and FMAs, a
  // register rotation) executed R times.  A fully unrolled triangle is
  // ~3x slower here -- a single warp streaming tens of KB of straight-line
  // code misses the instruction cache on every line.
  for (int k = 0; k < R; ++k) {
    const double piv = __shfl_sync(0xffffffffu, col[0], k);
    if (!(piv > 0.0)) {
      ok = false;
      break;
    }
    const double u = sqrt(piv);
    const double inv = 1.0 / u;
    const double ukb = lane == k ? u : (lane > k ? col[0] * inv : 0.0);
    if (lane >= k && lane < R) H[k * R + lane] = ukb;
    if (lane == 0) inv_diag[k] = inv;
#pragma unroll
    for (int a = 1; a < RB; ++a) {
      // U[k][k + a] from lane k + a (0 past the matrix)
      const int src = k + a;
      const double uka = __shfl_sync(0xffffffffu, ukb, src < 32 ? src : 31);
      if (src <= lane && src < R) col[a] = fma(-uka, ukb, col[a]);
    }
#pragma unroll
    for (int a = 0; a < RB - 1; ++a) col[a] = col[a + 1];
    col[RB - 1] = 0.0;
  }
  __syncwarp();
  if (lane == 0) *flag = ok ? 1 : 0;
}

// rank buckets up to RB (a kernel built for bucket RB only holds RB-sized
// register arrays)
template <int RB = kFastR>
__device__ __forceinline__ void warp_cholesky_fast_nosync(double* __restrict__ H, int R,
                                                          double* __restrict__ inv_diag,
                                                          int* flag) {
  if (RB <= 8 || R <= 8)
    warp_cholesky_rb<8>(H, R, inv_diag, flag);
  else if (RB <= 16 || R <= 16)
    warp_cholesky_rb<16>(H, R, inv_diag, flag);
  else if (RB <= 24 || R <= 24)
    warp_cholesky_rb<24>(H, R, inv_diag, flag);
  else
    warp_cholesky_rb<32>(H, R, inv_diag, flag);
}

__device__ inline bool warp_cholesky_fast(double* H, int R, double* inv_diag, int* flag) {
  if (threadIdx.x < 32) warp_cholesky_fast_nosync(H, R, inv_diag, flag);
  __syncthreads();
  return *flag != 0;
}

// Copy rows [0, cnt) of the R-wide column block at Mb (row stride ld) into
// Xs (pitch P; Xs == nullptr: check only).  Consecutive threads take
// consecutive elements of the block, so a warp's loads cover a few rows'
// contiguous R-double segments (coalesced) and four loads per thread are in
// flight at once.  Returns nonzero when any value is non-finite.
__device__ __forceinline__ int stage_block(const double* __restrict__ Mb, long long ld, int cnt, int R,
                                  int P, double* __restrict__ Xs, int t0, int nt) {
  int bad = 0;
  const int total = cnt * R;
  for (int e0 = t0; e0 < total; e0 += 4 * nt) {
    double v[4];
    int ii[4], aa[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * nt;
      ii[u] = e / R;
      aa[u] = e - ii[u] * R;
      v[u] = e < total ? Mb[(long long)ii[u] * ld + aa[u]] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      bad |= !isfinite(v[u]);
      if (Xs != nullptr && e0 + u * nt < total) Xs[ii[u] * P + aa[u]] = v[u];
    }
  }
  return bad;
}

// Gram of an existing column block (rows x R at F + off), chunked through Xs.
template <int RB = kFastR>
__device__ inline void block_gram_fast(const double* F, long long ld, int rows, int R, double* Xs,
                                       double* G) {
  const int P = fast_pitch(R);
  FastPairsT<fast_np(RB)> pr;
  pr.init(R);
  for (int base = 0; base < rows; base += kUpdThreads) {
    const int cnt = min(kUpdThreads, rows - base);
    stage_block(F + (long long)base * ld, ld, cnt, R, P, Xs, threadIdx.x, kUpdThreads);
    __syncthreads();
    pr.accumulate(Xs, P, cnt);
    __syncthreads();
  }
  pr.store(G, R);
}

// One row's two triangular solves (U^T y = m, then U x = y; dpotrs order,
// reciprocal diagonal) with the row in registers (rank bucket RB), so each
// step is a chain of one multiply and the independent FMAs of the remaining
// entries instead of shared-memory read-modify-writes.  Same operation order
// per entry as the shared-memory version (bitwise identical).
template <int RB>
__device__ __forceinline__ void solve_row_reg(double* __restrict__ xs,
                                              const double* __restrict__ U,
                                              const double* __restrict__ inv_diag, int R) {
  double x[RB];
#pragma unroll
  for (int a = 0; a < RB; ++a) x[a] = a < R ? xs[a] : 0.0;
#pragma unroll
  for (int k = 0; k < RB; ++k) {  // U^T y = m
    if (k < R) {
      const double yk = x[k] * inv_diag[k];
      x[k] = yk;
      const double* urow = U + k * R;
#pragma unroll
      for (int a = k + 1; a < RB; ++a)
        if (a < R) x[a] = fma(-urow[a], yk, x[a]);
    }
  }
#pragma unroll
  for (int k = RB - 1; k >= 0; --k) {  // U x = y
    if (k < R) {
      const double xk = x[k] * inv_diag[k];
      x[k] = xk;
#pragma unroll
      for (int a = 0; a < k; ++a) x[a] = fma(-U[a * R + k], xk, x[a]);
    }
  }
#pragma unroll
  for (int a = 0; a < RB; ++a)
    if (a < R) xs[a] = x[a];
}

template <int RB = kFastR>
__device__ __forceinline__ bool block_solve_gram_fast(const double* __restrict__ U,
                                             const double* __restrict__ inv_diag, int R,
                                             const double* __restrict__ Mb, long long ldm,
                                             int rows, double* __restrict__ A, long long lda,
                                             double* __restrict__ Xs, double* __restrict__ G,
                                             bool want_inner, double* inner, double* red,
                                             bool first_chunk_staged = false,
                                             long long* stamps = nullptr) {
  const int P = fast_pitch(R);
  FastPairsT<fast_np(RB)> pr;
  double dot = 0.0;
  int bad = 0;
  for (int base = 0; base < rows; base += kUpdThreads) {
    const int cnt = min(kUpdThreads, rows - base);
    const double* Mc = Mb + (long long)base * ldm;
    if (base > 0 || !first_chunk_staged) {
      stage_block(Mc, ldm, cnt, R, P, Xs, threadIdx.x, kUpdThreads);
      __syncthreads();
    }
    if (threadIdx.x < cnt) {
      double* x = Xs + threadIdx.x * P;
      if (RB <= 8 || R <= 8)
        solve_row_reg<8>(x, U, inv_diag, R);
      else if (RB <= 16 || R <= 16)
        solve_row_reg<16>(x, U, inv_diag, R);
      else if (RB <= 24 || R <= 24)
        solve_row_reg<24>(x, U, inv_diag, R);
      else
        solve_row_reg<32>(x, U, inv_diag, R);
    }
    __syncthreads();
    if (stamps && threadIdx.x == 32) stamps[0] = clock64();
    double* Ac = A + (long long)base * lda;
    const int total = cnt * R;
    for (int e = threadIdx.x; e < total; e += kUpdThreads) {
      const int i = e / R, a = e - i * R;
      const double v = Xs[i * P + a];
      bad |= !isfinite(v);
      Ac[(long long)i * lda + a] = v;
      if (want_inner) dot = fma(v, Mc[(long long)i * ldm + a], dot);
    }
    if (stamps && threadIdx.x == 32) stamps[1] = clock64();
    if (base == 0) pr.init(R);  // not live across the first chunk's solve
    pr.accumulate(Xs, P, cnt);
    __syncthreads();
    if (stamps && threadIdx.x == 32) stamps[2] = clock64();
  }
  if (__syncthreads_or(bad)) return false;
  pr.store(G, R);
  if (want_inner) *inner = block_sum(dot, red);
  return true;
}

}  // namespace cals
