// Non-negative factor rows: warm-started Lawson-Hanson active-set search, one
// warp per factor row (R <= 32, lane a owns variable a).  Restates
// pkg/src/cals/als.py:185-263 (nnls_solve_row) and als.py:266-278
// (nnls_update); the passive-set systems are solved by LU with partial
// pivoting (dgesv, as np.linalg.solve) with an eigen-pinv least-squares
// fallback for an exactly singular pivot (np.linalg.lstsq).
#pragma once

#include "common.cuh"
#include "update.cuh"

namespace cals {

constexpr int kNnlsP = 33;  // smem row pitch of the per-warp p x p system

__device__ __forceinline__ unsigned lane_mask_below(int lane) { return (1u << lane) - 1u; }

// z[P] = solve(H[P,P], f[P]), z = 0 off P.  `Ws` is this warp's scratch:
// kNnlsP * 32 doubles for the system + 32 for the RHS + 32 * 32 for a pinv
// fallback eigenbasis.  Returns this lane's z.
__device__ inline double nnls_solve_passive(const double* H, int R, unsigned P, double f_lane,
                                            double* Ws) {
  const int lane = threadIdx.x & 31;
  const int p = __popc(P);
  if (p == 0) return 0.0;
  __syncwarp();  // the previous solve's lanes are done reading A / b
  double* A = Ws;                    // [p][kNnlsP]
  double* b = Ws + kNnlsP * 32;      // [32]
  const bool in = lane < R && ((P >> lane) & 1u);
  const int pos = __popc(P & lane_mask_below(lane));  // compressed index of this lane
  // gather H[P,P] (lane = compressed row) and f[P]
  {
    int src = -1, cnt = 0;
    for (int a = 0; a < R; ++a)
      if ((P >> a) & 1u) {
        if (cnt == lane) src = a;
        ++cnt;
      }
    if (lane < p) {
      int cj = 0;
      for (int a = 0; a < R; ++a)
        if ((P >> a) & 1u) A[lane * kNnlsP + cj++] = H[src * R + a];
    }
    if (in) b[pos] = f_lane;
  }
  __syncwarp();
  // LU with partial pivoting (dgetf2: first max |pivot|, reciprocal scaling)
  bool singular = false;
  int perm_of_lane = lane;  // row currently held at position `lane`
  for (int k = 0; k < p; ++k) {
    double v = (lane >= k && lane < p) ? fabs(A[lane * kNnlsP + k]) : -1.0;
    int arg = lane;
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v, o);
      const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
      if (ov > v || (ov == v && oa < arg)) {
        v = ov;
        arg = oa;
      }
    }
    if (!(v > 0.0)) {
      singular = true;
      break;
    }
    if (arg != k) {  // swap rows k and arg (and the RHS)
      for (int j = lane; j < p; j += 32) {
        const double t = A[k * kNnlsP + j];
        A[k * kNnlsP + j] = A[arg * kNnlsP + j];
        A[arg * kNnlsP + j] = t;
      }
      if (lane == 0) {
        const double t = b[k];
        b[k] = b[arg];
        b[arg] = t;
      }
      const int pk = __shfl_sync(0xffffffffu, perm_of_lane, k);
      const int pa = __shfl_sync(0xffffffffu, perm_of_lane, arg);
      if (lane == k) perm_of_lane = pa;
      if (lane == arg) perm_of_lane = pk;
    }
    __syncwarp();
    const double rinv = 1.0 / A[k * kNnlsP + k];
    if (lane > k && lane < p) {
      const double l = A[lane * kNnlsP + k] * rinv;
      A[lane * kNnlsP + k] = l;
      // a_ij - l_ik u_kj with two roundings, as OpenBLAS's dgetf2 (dot of
      // length one, then the subtraction): with the reciprocal multiplier
      // and the fused forward / back substitutions this reproduces
      // np.linalg.solve bit for bit on 2 x 2 systems (the reference suite's
      // exact enumeration check, test_acceptance.py:183-188)
      for (int j = k + 1; j < p; ++j)
        A[lane * kNnlsP + j] =
            __dsub_rn(A[lane * kNnlsP + j], __dmul_rn(l, A[k * kNnlsP + j]));
    }
    __syncwarp();
  }
  double zc = 0.0;  // solution in compressed index `lane`
  if (!singular) {
    // forward (unit lower), then back (upper) -- serial over rows, lane 0
    if (lane == 0) {
      for (int i = 0; i < p; ++i) {
        double s = b[i];
        for (int j = 0; j < i; ++j) s = fma(-A[i * kNnlsP + j], b[j], s);
        b[i] = s;
      }
      for (int i = p - 1; i >= 0; --i) {
        double s = b[i];
        for (int j = i + 1; j < p; ++j) s = fma(-A[i * kNnlsP + j], b[j], s);
        b[i] = s / A[i * kNnlsP + i];
      }
    }
    __syncwarp();
    zc = lane < p ? b[lane] : 0.0;
  } else {
    // lstsq fallback: minimum-norm solution through the eigenbasis of the
    // (symmetric) system, cutoff eps * p * lambda_max (np.linalg.lstsq rcond)
    double* V = Ws + kNnlsP * 32 + 32;
    if (lane < p) {
      int cj = 0, src = -1, cnt = 0;
      for (int a = 0; a < R; ++a)
        if ((P >> a) & 1u) {
          if (cnt == lane) src = a;
          ++cnt;
        }
      for (int a = 0; a < R; ++a)
        if ((P >> a) & 1u) A[lane * p + cj++] = H[src * R + a];
    }
    if (in) b[pos] = f_lane;
    __syncwarp();
    // pack A densely as p x p for warp_jacobi
    warp_jacobi(A, V, p);
    __syncwarp();
    double lmax = 0.0;
    for (int k = 0; k < p; ++k) lmax = fmax(lmax, fabs(A[k * p + k]));
    const double cut = 2.220446049250313e-16 * p * lmax;
    if (lane < p) {
      double s = 0.0;
      for (int k = 0; k < p; ++k) {
        const double lk = A[k * p + k];
        if (fabs(lk) > cut) {
          double proj = 0.0;
          for (int j = 0; j < p; ++j) proj = fma(V[j * p + k], b[j], proj);
          s = fma(V[lane * p + k], proj / lk, s);
        }
      }
      zc = s;
    }
    __syncwarp();
  }
  // scatter back: lane a takes compressed entry pos(a)
  const double z = __shfl_sync(0xffffffffu, zc, in ? pos : 0);
  (void)perm_of_lane;
  return in ? z : 0.0;
}

// One row: returns x (this lane's entry), updates *active (bit set = pinned
// to zero), *converged.
__device__ inline double nnls_row(const double* H, int R, double f_lane, unsigned* active,
                                  bool* converged, double* Ws, int max_iter_in = -1) {
  const int lane = threadIdx.x & 31;
  const unsigned full = R == 32 ? 0xffffffffu : ((1u << R) - 1u);
  const bool valid = lane < R;
  unsigned passive = ~(*active) & full;
  double scale = valid ? fabs(f_lane) : 0.0;
  for (int o = 16; o > 0; o >>= 1) scale = fmax(scale, __shfl_xor_sync(0xffffffffu, scale, o));
  const double tol = 1e-11 * fmax(scale, 1e-300);
  const int max_iter = max_iter_in >= 0 ? max_iter_in : 3 * R;
  double x = 0.0;
  int steps = 0;
  *converged = true;
  double z = nnls_solve_passive(H, R, passive, f_lane, Ws);
  while (true) {
    // restore feasibility of the passive solve (inner loop)
    while (true) {
      const bool inp = valid && ((passive >> lane) & 1u);
      const unsigned badm = __ballot_sync(0xffffffffu, inp && z <= 0.0);
      if (passive == 0u || badm == 0u) break;
      if (++steps > max_iter) {
        *converged = false;
        x = fmax(x, 0.0);
        if (!((passive >> lane) & 1u)) x = 0.0;
        *active = ~passive & full;
        return valid ? x : 0.0;
      }
      double ratio = INFINITY;
      if ((badm >> lane) & 1u) {
        const double denom = __dsub_rn(x, z);
        ratio = denom > 0.0 ? x / denom : 0.0;
      }
      for (int o = 16; o > 0; o >>= 1) ratio = fmin(ratio, __shfl_xor_sync(0xffffffffu, ratio, o));
      const double alpha = ratio;
      x = __dadd_rn(x, __dmul_rn(alpha, __dsub_rn(z, x)));
      const unsigned drop = __ballot_sync(0xffffffffu, inp && x <= tol);
      passive &= ~drop;
      if (!((passive >> lane) & 1u)) x = 0.0;
      z = nnls_solve_passive(H, R, passive, f_lane, Ws);
    }
    x = z;
    // KKT: w = f - H x, largest w over the zeroed variables
    double hx = 0.0;
    for (int b = 0; b < R; ++b) {
      const double xb = __shfl_sync(0xffffffffu, x, b);
      if (valid) hx = fma(H[lane * R + b], xb, hx);
    }
    double w = (valid && !((passive >> lane) & 1u)) ? __dsub_rn(f_lane, hx) : -INFINITY;
    int arg = lane;
    for (int o = 16; o > 0; o >>= 1) {  // argmax, first index on ties (np.argmax)
      const double ow = __shfl_xor_sync(0xffffffffu, w, o);
      const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
      if (ow > w || (ow == w && oa < arg)) {
        w = ow;
        arg = oa;
      }
    }
    if (w <= tol) break;
    if (++steps > max_iter) {
      *converged = false;
      break;
    }
    passive |= 1u << arg;
    z = nnls_solve_passive(H, R, passive, f_lane, Ws);
  }
  x = fmax(x, 0.0);
  if (!((passive >> lane) & 1u)) x = 0.0;
  *active = ~passive & full;
  return valid ? x : 0.0;
}

// Standalone rows (nnls_update / nnls_solve_row API): one warp per row of the
// rows x R block m (row-major, ldm); H is R x R (global); active[i] in/out.
__global__ void nnls_rows_kernel(int rows, int R, const double* __restrict__ m, long long ldm,
                                 const double* __restrict__ Hg, unsigned* active, double* x,
                                 long long ldx, int* conv, int max_iter) {
  extern __shared__ __align__(16) double sm[];
  double* H = sm;
  for (int idx = threadIdx.x; idx < R * R; idx += blockDim.x) H[idx] = Hg[idx];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  double* Ws = sm + R * R + warp * (kNnlsP * 32 + 32 + 32 * 32);
  for (int i = blockIdx.x * nw + warp; i < rows; i += gridDim.x * nw) {
    const double f = lane < R ? m[(long long)i * ldm + lane] : 0.0;
    unsigned act = active[i];
    bool ok = true;
    const double v = nnls_row(H, R, f, &act, &ok, Ws, max_iter);
    if (lane < R) x[(long long)i * ldx + lane] = v;
    if (lane == 0) {
      active[i] = act;
      conv[i] = ok ? 1 : 0;
    }
  }
}

}  // namespace cals
