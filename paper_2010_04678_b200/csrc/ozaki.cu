// Host side of the Ozaki-sliced INT8 tensor-core MTTKRP (see ozaki.cuh):
// per-tensor X slices (built once per tensor view), per-call Lo slices, and
// the launch that replaces the DMMA contraction of mttkrp.cu.
#include <cstdlib>
#include <cstring>

#include "internal.h"
#include "mttkrp.cuh"
#include "ozaki.cuh"

namespace cals {

using namespace oz;

// X slices of one 3-D view: xs[7][Dq][M][Kp] (int8 bit patterns), rex[Dq][M] =
// scale exponent ex per row (q, m).  Element (m, p, q) lives at x[m*sm + p*sp + q*sq].
// Block = 256 threads for rows m0..m0+31 of slab q; padded p in [Dp, Kp) -> 0.
__global__ void oz_slice_rows_kernel(const double* __restrict__ x, long long sm, long long sp,
                                     long long sq, int M, int Dp, int Kp, int Dq,
                                     uint8_t* __restrict__ xs, int* __restrict__ rex,
                                     int* __restrict__ out_of_range) {
  __shared__ double tile[32][33];
  __shared__ double red[8][33];
  __shared__ int ex[32];
  const int q = blockIdx.y, m0 = blockIdx.x * 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const double* xq = x + (long long)q * sq;
  const bool mfast = sm == 1;  // m contiguous in memory -> lanes along m
  // ---- pass 1: per-row max |x|
  if (mfast) {
    const int m = m0 + lane;
    double mx = 0.0;
    if (m < M)
      for (int p = w; p < Dp; p += 8) mx = fmax(mx, abs_or_inf(xq[m + (long long)p * sp]));
    red[w][lane] = mx;
    __syncthreads();
    if (w == 0) {
      double v = red[0][lane];
#pragma unroll
      for (int k = 1; k < 8; ++k) v = fmax(v, red[k][lane]);
      red[0][lane] = v;
    }
  } else {
    for (int r = w; r < 32; r += 8) {
      const int m = m0 + r;
      double v = 0.0;
      if (m < M)
        for (int p = lane; p < Dp; p += 32)
          v = fmax(v, abs_or_inf(xq[(long long)m * sm + (long long)p * sp]));
#pragma unroll
      for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
      if (lane == 0) red[0][r] = v;
    }
  }
  __syncthreads();
  if (w == 0) {
    const int e = scale_exp_checked(red[0][lane]);
    ex[lane] = e;
    const int m = m0 + lane;
    if (m < M) {
      rex[(long long)q * M + m] = e;
      // the epilogue scales by exponent-field adds: keep |ex| <= 900; a
      // non-finite tensor entry sends the whole view to the DMMA kernel
      if (e == kNonFinite || e < -900 || e > 900) atomicOr(out_of_range, 1);
    }
  }
  __syncthreads();
  // ---- pass 2: slices, written p-contiguous (32-byte segments per warp store)
  const size_t slice_stride = size_t(Dq) * size_t(M) * size_t(Kp);
  // dynamic-range guard: per row, nonzero entries and those below
  // 2^-kRangeBits of the row maximum (rows r = w, w + 8, w + 16, w + 24)
  int n_nz[4] = {0, 0, 0, 0}, n_small[4] = {0, 0, 0, 0};
  double thr[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int e = ex[w + 8 * j];
    thr[j] = (e == kNonFinite) ? 0.0 : ldexp(1.0, e - kRangeBits);
  }
  for (int p0 = 0; p0 < Kp; p0 += 32) {
    if (mfast) {
      const int m = m0 + lane;
      for (int pp = w; pp < 32; pp += 8) {
        const int p = p0 + pp;
        tile[lane][pp] = (m < M && p < Dp) ? xq[m + (long long)p * sp] : 0.0;
      }
    } else {
      const int p = p0 + lane;
      for (int r = w; r < 32; r += 8) {
        const int m = m0 + r;
        tile[r][lane] = (m < M && p < Dp) ? xq[(long long)m * sm + (long long)p * sp] : 0.0;
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = w + 8 * j;
      const int m = m0 + r;
      if (m >= M) continue;
      const double v = tile[r][lane];
      const double a = fabs(v);
      n_nz[j] += a != 0.0;
      n_small[j] += a != 0.0 && a < thr[j];
      uint8_t s[kSlices];
      slice7(v, ex[r], s);
      uint8_t* dst = xs + (size_t(q) * M + m) * size_t(Kp) + p0 + lane;
#pragma unroll
      for (int k = 0; k < kSlices; ++k) dst[k * slice_stride] = s[k];
    }
    __syncthreads();
  }
  // view-wide dynamic-range census (ozaki_check): nonzero entries, and those
  // kept with fewer than 55 - kRangeBits bits (below 2^-kRangeBits of their
  // row maximum)
  int nz = 0, nsmall = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (m0 + w + 8 * j < M) {
      nz += n_nz[j];
      nsmall += n_small[j];
    }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    nz += __shfl_xor_sync(0xffffffffu, nz, o);
    nsmall += __shfl_xor_sync(0xffffffffu, nsmall, o);
  }
  if (lane == 0 && nz > 0) {
    unsigned long long* census = reinterpret_cast<unsigned long long*>(out_of_range + 2);
    atomicAdd(census, (unsigned long long)nsmall);
    atomicAdd(census + 1, (unsigned long long)nz);
  }
}

// Single-pass version of oz_slice_rows_kernel for views whose 32-row block
// fits in shared memory (Kp <= kRowsTileMaxKp): the block's 32 rows x Kp
// values are loaded once into tile[p][33] with every load of a thread in
// flight (the two-pass kernel reads the tensor twice with a dependent chain
// of loads per thread and moves ~1.1 TB/s), the row maxima come from the same
// loads, and the slices are written from the tile.  Same exponents, slices
// and dynamic-range census as oz_slice_rows_kernel.
constexpr int kRowsTileMaxKp = 384;
__global__ void __launch_bounds__(256) oz_slice_rows_tile_kernel(
    const double* __restrict__ x, long long sm, long long sp, long long sq, int M, int Dp, int Kp,
    int Dq, uint8_t* __restrict__ xs, int* __restrict__ rex, int* __restrict__ out_of_range) {
  extern __shared__ double tile[];  // [Kp][33]
  __shared__ double red[8][33];
  __shared__ int ex[32];
  const int q = blockIdx.y, m0 = blockIdx.x * 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const double* xq = x + (long long)q * sq;
  if (sm == 1) {  // m contiguous: lanes along m, warps stride p
    const int m = m0 + lane;
    const bool mv = m < M;
    double mx = 0.0;
    int p = w;
    for (; p + 8 * 7 < Kp; p += 8 * 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int pu = p + 8 * u;
        v[u] = (mv && pu < Dp) ? xq[m + (long long)pu * sp] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        mx = fmax(mx, abs_or_inf(v[u]));
        tile[(p + 8 * u) * 33 + lane] = v[u];
      }
    }
    for (; p < Kp; p += 8) {
      const double v = (mv && p < Dp) ? xq[m + (long long)p * sp] : 0.0;
      mx = fmax(mx, abs_or_inf(v));
      tile[p * 33 + lane] = v;
    }
    red[w][lane] = mx;
    __syncthreads();
    if (w == 0) {
      double v = red[0][lane];
#pragma unroll
      for (int k = 1; k < 8; ++k) v = fmax(v, red[k][lane]);
      red[0][lane] = v;
    }
  } else {  // p contiguous: lanes along p, warps take rows
    for (int r = w; r < 32; r += 8) {
      const int m = m0 + r;
      const bool mv = m < M;
      const double* row = xq + (long long)m * sm;
      double mx = 0.0;
      int p = lane;
      for (; p + 32 * 3 < Kp; p += 32 * 4) {
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int pu = p + 32 * u;
          v[u] = (mv && pu < Dp) ? row[(long long)pu * sp] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          mx = fmax(mx, abs_or_inf(v[u]));
          tile[(p + 32 * u) * 33 + r] = v[u];
        }
      }
      for (; p < Kp; p += 32) {
        const double v = (mv && p < Dp) ? row[(long long)p * sp] : 0.0;
        mx = fmax(mx, abs_or_inf(v));
        tile[p * 33 + r] = v;
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (lane == 0) red[0][r] = mx;
    }
  }
  __syncthreads();
  if (w == 0) {
    const int e = scale_exp_checked(red[0][lane]);
    ex[lane] = e;
    const int m = m0 + lane;
    if (m < M) {
      rex[(long long)q * M + m] = e;
      if (e == kNonFinite || e < -900 || e > 900) atomicOr(out_of_range, 1);
    }
  }
  __syncthreads();
  const size_t slice_stride = size_t(Dq) * size_t(M) * size_t(Kp);
  int nz = 0, nsmall = 0;
  for (int r = w; r < 32; r += 8) {
    const int m = m0 + r;
    if (m >= M) continue;
    const int e = ex[r];
    const double thr = (e == kNonFinite) ? 0.0 : ldexp(1.0, e - kRangeBits);
    uint8_t* row = xs + (size_t(q) * M + m) * size_t(Kp);
    for (int p = lane; p < Kp; p += 32) {
      const double v = tile[p * 33 + r];
      const double a = fabs(v);
      nz += a != 0.0;
      nsmall += a != 0.0 && a < thr;
      uint8_t sl[kSlices];
      slice7(v, e, sl);
#pragma unroll
      for (int k = 0; k < kSlices; ++k) row[p + k * slice_stride] = sl[k];
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    nz += __shfl_xor_sync(0xffffffffu, nz, o);
    nsmall += __shfl_xor_sync(0xffffffffu, nsmall, o);
  }
  if (lane == 0 && nz > 0) {
    unsigned long long* census = reinterpret_cast<unsigned long long*>(out_of_range + 2);
    atomicAdd(census, (unsigned long long)nsmall);
    atomicAdd(census + 1, (unsigned long long)nz);
  }
}

// Lo slices: ls[7][cap_pad][Kp] (column c of lo as a p-contiguous row),
// cex[c] = scale exponent el of column c.  Block (x, y) = 256 threads for
// columns 32x..32x+31 and p-chunk y (32 values); the column max is taken
// over all p by every chunk's block (L2-resident, 8 loads per thread).
__global__ void oz_slice_cols_kernel(const double* __restrict__ lo, long long ld, int Dp, int Kp,
                                     const int* width_ptr, int width, long long cap_pad,
                                     uint8_t* __restrict__ ls, int* __restrict__ cex,
                                     int* __restrict__ queue, const int* __restrict__ stale) {
  __shared__ double tile[32][33];
  __shared__ double red[8][33];
  __shared__ int ex[32];
  griddep_wait();  // launched with PDL (launch_dep): predecessors complete
  // the contraction kernel that follows claims its work units from *queue
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *queue = 0;
  if (stale && *stale == 0) return;  // the solve kernel already wrote these slices
  const int W = width_ptr ? *width_ptr : width;
  const int c0 = blockIdx.x * 32, p0 = blockIdx.y * 32;
  if (c0 >= W) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = c0 + lane;
  {
    // One pass over the column block: up to 32 loads in flight per thread
    // (a rolled loop waits one L2 round trip per row), the column max (order
    // independent) and, for the rows of this block's p-chunk, the tile.
    for (int pp = w; pp < 32; pp += 8) tile[pp][lane] = 0.0;
    double mx = 0.0;
    if (c < W) {
      for (int pb = w; pb < Dp; pb += 8 * 32) {
        double v[32];
#pragma unroll
        for (int u = 0; u < 32; ++u) {
          const int p = pb + 8 * u;
          v[u] = p < Dp ? lo[(long long)p * ld + c] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 32; ++u) {
          const int p = pb + 8 * u;
          mx = fmax(mx, abs_or_inf(v[u]));
          if (p >= p0 && p < p0 + 32 && p < Dp) tile[p - p0][lane] = v[u];
        }
      }
    }
    red[w][lane] = mx;
  }
  __syncthreads();
  if (w == 0) {
    double v = red[0][lane];
#pragma unroll
    for (int k = 1; k < 8; ++k) v = fmax(v, red[k][lane]);
    const int e = scale_exp_checked(v);
    ex[lane] = e;
    if (blockIdx.y == 0 && c < W) cex[c] = e;
  }
  __syncthreads();
  const size_t slice_stride = size_t(cap_pad) * size_t(Kp);
  for (int cc = w; cc < 32; cc += 8) {
    uint8_t sl[kSlices];
    slice7(tile[lane][cc], ex[cc], sl);
    uint8_t* dst = ls + size_t(c0 + cc) * size_t(Kp) + p0 + lane;
#pragma unroll
    for (int k = 0; k < kSlices; ++k) dst[k * slice_stride] = sl[k];
  }
}

// Short contractions (Kp <= 256): one block per 32 columns does the whole
// column block -- one pass of loads (<= 32 per thread, all in flight) into a
// shared-memory tile, the column max from the same values, then every
// (column, p) element sliced -- instead of Kp/32 blocks that each re-read the
// full columns for the max.  Same slices and exponents as
// oz_slice_cols_kernel.
constexpr int kColsAllMaxKp = 256;
__global__ void __launch_bounds__(256) oz_slice_cols_all_kernel(
    const double* __restrict__ lo, long long ld, int Dp, int Kp, const int* width_ptr, int width,
    long long cap_pad, uint8_t* __restrict__ ls, int* __restrict__ cex, int* __restrict__ queue,
    const int* __restrict__ stale) {
  extern __shared__ double ctile[];  // [Kp][33]
  __shared__ double red[8][33];
  __shared__ int ex[32];
  griddep_wait();  // launched with PDL (launch_dep): predecessors complete
  if (blockIdx.x == 0 && threadIdx.x == 0) *queue = 0;
  if (stale && *stale == 0) return;  // the solve kernel already wrote these slices
  const int W = width_ptr ? *width_ptr : width;
  const int c0 = blockIdx.x * 32;
  if (c0 >= W) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = c0 + lane;
  double v[kColsAllMaxKp / 8];
#pragma unroll
  for (int u = 0; u < kColsAllMaxKp / 8; ++u) {
    const int p = w + 8 * u;
    v[u] = (c < W && p < Dp) ? lo[(long long)p * ld + c] : 0.0;
  }
  double mx = 0.0;
#pragma unroll
  for (int u = 0; u < kColsAllMaxKp / 8; ++u) {
    const int p = w + 8 * u;
    mx = fmax(mx, abs_or_inf(v[u]));
    if (p < Kp) ctile[p * 33 + lane] = v[u];
  }
  red[w][lane] = mx;
  __syncthreads();
  if (w == 0) {
    double m = red[0][lane];
#pragma unroll
    for (int k = 1; k < 8; ++k) m = fmax(m, red[k][lane]);
    const int e = scale_exp_checked(m);
    ex[lane] = e;
    if (c < W) cex[c] = e;
  }
  __syncthreads();
  const size_t slice_stride = size_t(cap_pad) * size_t(Kp);
  for (int idx = threadIdx.x; idx < 32 * Kp; idx += blockDim.x) {
    const int cc = idx / Kp, p = idx - cc * Kp;  // consecutive threads: consecutive p
    uint8_t sl[kSlices];
    slice7(ctile[p * 33 + cc], ex[cc], sl);
    uint8_t* dst = ls + size_t(c0 + cc) * size_t(Kp) + p;
#pragma unroll
    for (int k = 0; k < kSlices; ++k) dst[k * slice_stride] = sl[k];
  }
}

static int view_strides(const Tensor& t, const ModePlan& p, long long& sm, long long& sp,
                        long long& sq) {
  const long long s0 = 1, s1 = p.D[0], s2 = p.D[0] * p.D[1];
  switch (p.role) {
    case kRoleFirst: sm = s0; sp = s1; sq = s2; break;    // (m, p, q)
    case kRoleFirstQP: sm = s0; sq = s1; sp = s2; break;  // (m, q, p)
    case kRoleMiddle: sp = s0; sm = s1; sq = s2; break;   // (p, m, q)
    case kRoleLast: sp = s0; sq = s1; sm = s2; break;     // (p, q, m)
    default: return kErrInvalid;
  }
  (void)t;
  return kOk;
}

static long long kp_of(long long Dp) { return (Dp + KSTEP - 1) / KSTEP * KSTEP; }

constexpr size_t kFlagBytes = 24;

// Dynamic-range guard of the tensor slices (see oz_slice_rows_kernel);
// CALS_OZ_RANGE_GUARD=0 disables it (tests of the raw INT8 envelope).
bool ozaki_range_guard() {
  static const bool on = [] {
    const char* env = getenv("CALS_OZ_RANGE_GUARD");
    return !(env && strcmp(env, "0") == 0);
  }();
  return on;
}

bool ozaki_enabled() {
  static const bool on = [] {
    const char* env = getenv("CALS_MTTKRP");
    return !(env && (strcmp(env, "dmma") == 0 || strcmp(env, "0") == 0));
  }();
  return on;
}

// The INT8 path pays off when the tensor-core work per slab (K = Dp) is large
// against the per-slab epilogue and the 64-row m-tiles are well filled
// (measured: 200^3 1.23x, 500^3 2.2x faster than DMMA; an EEM mode with
// M = 21 output rows is faster on DMMA).  CALS_MTTKRP=ozaki forces it for
// every eligible shape, CALS_MTTKRP=dmma disables it.
bool ozaki_eligible(const ModePlan& p) {
  if (!ozaki_enabled() || p.role < 0 || p.role > 3 || kp_of(p.Dp) > 2048 || p.M < 1 ||
      p.Dq < 1 || p.Dq > 65535)
    return false;
  static const bool force = [] {
    const char* env = getenv("CALS_MTTKRP");
    return env && strcmp(env, "ozaki") == 0;
  }();
  if (force) return true;
  const double m_fill = double(p.M) / double((p.M + BNM - 1) / BNM * BNM);
  const double k_fill = double(p.Dp) / double(kp_of(p.Dp));
  // >= 3 slabs per split: the per-unit pipeline fill and the per-slab
  // epilogue must amortise over enough tensor-core work; views with few slabs
  // (Dq < 64, e.g. the EEM's 21) take ~2 per split instead (plan_splits
  // picks S = ceil(Dq / 2) for them; c3: 11 splits, 1.09x over DMMA)
  const bool slabs_ok = p.Dq >= 3LL * p.S || (p.Dq < 64 && 2LL * p.S <= p.Dq + 1);
  return p.Dp >= 128 && m_fill * k_fill >= 0.6 && slabs_ok;
}

// m tiling (see Args): full 64-row tiles plus, when the M % 64 leftover rows
// of a q-split's slabs fit one tile, a packed remainder tile per split
struct MTiling {
  int tm_full, rem_rows, rem_slabs;
};
static MTiling m_tiling(const ModePlan& p) {
  const long long r = p.M % BNM, nslab = (p.Dq + p.S - 1) / p.S;
  if (r > 0 && r * nslab <= BNM) return {int(p.M / BNM), int(r), int(nslab)};
  return {int((p.M + BNM - 1) / BNM), 0, 0};
}

// Split count for an INT8 view (shape only): among 24..48 splits, the one
// minimising the 64-row tile passes (the packed remainder tile is one pass per
// split, and only packs when M % 64 rows x slabs per split fit 64 columns)
// plus the split reduction's traffic (S partial blocks, ~49 / (Dq Kp) of the
// contraction time each, measured at c2).  c2 (200^3): 25 splits, 8 slabs
// each, the 8 leftover rows of a split fill a whole remainder tile (625 instead
// of 632 passes per column tile, 25 instead of 32 partials).  Views where no
// count packs better keep the default.
int ozaki_refine_splits(const ModePlan& base) {
  auto passes = [&](int S) {
    ModePlan q = base;
    q.S = S;
    const MTiling mt = m_tiling(q);
    return double(mt.tm_full) * double(q.Dq) + (mt.rem_rows ? double(S) : 0.0);
  };
  const double kp = double(kp_of(base.Dp));
  auto cost = [&](int S) { return passes(S) * (1.0 + 49.0 * S / (double(base.Dq) * kp)); };
  const double p0 = passes(base.S);
  int best = base.S;
  double best_cost = cost(base.S);
  for (int S = 24; S <= 48 && 3LL * S <= base.Dq; ++S) {
    if (passes(S) > 0.995 * p0) continue;  // only a real packing gain moves it
    const double c = cost(S);
    if (c < best_cost) {
      best_cost = c;
      best = S;
    }
  }
  return best;
}

// 28 slice products x 2 ops per MAC over the padded tiles the kernel runs
double ozaki_tensor_ops(const ModePlan& p, long long width) {
  const MTiling mt = m_tiling(p);
  const double wp = double((width + BMC - 1) / BMC * BMC);
  const double tile_passes = double(mt.tm_full) * double(p.Dq) + (mt.rem_rows ? double(p.S) : 0.0);
  return 2.0 * 28.0 * double(BNM) * tile_passes * wp * double(kp_of(p.Dp));
}

size_t ozaki_ws_bytes(const ModePlan& p, long long cap) {
  const long long cap_pad = (cap + BMC - 1) / BMC * BMC;
  return size_t(kSlices) * size_t(cap_pad) * size_t(kp_of(p.Dp)) + size_t(cap_pad) * 8 + 1024;
}

// A view whose slicing found rows beyond 2^+-900 or a non-finite entry is
// dropped (it stays on DMMA), and so is one where most nonzero entries sit
// more than 2^kRangeBits below their row maximum (they would keep fewer than
// 55 - kRangeBits bits; CALS_OZ_RANGE_GUARD=0 keeps such views on INT8).  The
// check reads the device flag block: done here when `validate`, else deferred
// to ozaki_validate (so the slicing can overlap host work, e.g. the pool
// packing of run()).
static int ozaki_check(Tensor& t, int key, OzSlices& o, cudaStream_t stream, bool* keep) {
  int h[kFlagBytes / 4] = {0};
  CALS_CUDA_TRY(cudaMemcpyAsync(h, o.flag, kFlagBytes, cudaMemcpyDeviceToHost, stream));
  CALS_CUDA_TRY(cudaStreamSynchronize(stream));
  CALS_CUDA_TRY(cudaFreeAsync(o.flag, stream));
  o.flag = nullptr;
  unsigned long long census[2];
  memcpy(census, h + 2, sizeof(census));
  const bool coarse = ozaki_range_guard() && 2 * census[0] > census[1];
  *keep = h[0] == 0 && !coarse;
  if (!*keep) {
    cudaFreeAsync(o.xs, stream);
    cudaFreeAsync(o.rex, stream);
  }
  (void)t;
  (void)key;
  return kOk;
}

int ozaki_validate(Tensor& t, int key, cudaStream_t stream) {
  std::lock_guard<std::mutex> lk(t.mu);
  auto it = t.oz.find(key);
  if (it == t.oz.end() || !it->second.flag) return kOk;
  bool keep = true;
  const int rc = ozaki_check(t, key, it->second, stream, &keep);
  if (rc) return rc;
  if (!keep) t.oz.erase(it);
  return kOk;
}

int ozaki_prepare(Tensor& t, const ModePlan& p, int key, cudaStream_t stream, bool validate) {
  if (!ozaki_eligible(p)) return kOk;
  {
    std::unique_lock<std::mutex> lk(t.mu);
    if (t.oz.count(key)) {
      lk.unlock();
      return validate ? ozaki_validate(t, key, stream) : kOk;
    }
  }
  long long sm, sp, sq;
  if (view_strides(t, p, sm, sp, sq)) return kOk;
  OzSlices o{};
  o.Kp = kp_of(p.Dp);
  o.M = p.M;
  o.Dq = p.Dq;
  o.Dp = p.Dp;
  const size_t xs_bytes = size_t(kSlices) * size_t(p.Dq) * size_t(p.M) * size_t(o.Kp);
  {
    // too large for a third of the device: this view stays on DMMA
    static const size_t total = [] {
      size_t f = 0, tot = 0;
      return cudaMemGetInfo(&f, &tot) == cudaSuccess ? tot : size_t(0);
    }();
    if (xs_bytes > total / 3) return kOk;
  }
  CALS_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&o.xs), xs_bytes, stream));
  poison_alloc(o.xs, xs_bytes, stream, true);
  CALS_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&o.rex), size_t(p.Dq) * p.M * 4, stream));
  poison_alloc(o.rex, size_t(p.Dq) * p.M * 4, stream, true);
  int* flag = nullptr;
  // [0] out-of-range / non-finite flag, [2..5] two u64 census counters
  CALS_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&flag), kFlagBytes, stream));
  CALS_CUDA_TRY(cudaMemsetAsync(flag, 0, kFlagBytes, stream));
  dim3 grid((unsigned)((p.M + 31) / 32), (unsigned)p.Dq);
  static const bool tile_ok = [] {  // CALS_OZ_ROWS_TILE=0: two-pass kernel (A/B)
    const char* env = getenv("CALS_OZ_ROWS_TILE");
    return !(env && strcmp(env, "0") == 0);
  }();
  if (tile_ok && o.Kp <= kRowsTileMaxKp) {
    const size_t smem = size_t(o.Kp) * 33 * 8;
    static std::once_flag once;
    static cudaError_t attr = cudaSuccess;
    std::call_once(once, [] {
      attr = cudaFuncSetAttribute(oz_slice_rows_tile_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kRowsTileMaxKp * 33 * 8);
    });
    CALS_CUDA_TRY(attr);
    oz_slice_rows_tile_kernel<<<grid, 256, smem, stream>>>(t.data, sm, sp, sq, (int)p.M,
                                                           (int)p.Dp, (int)o.Kp, (int)p.Dq, o.xs,
                                                           o.rex, flag);
  } else {
    oz_slice_rows_kernel<<<grid, 256, 0, stream>>>(t.data, sm, sp, sq, (int)p.M, (int)p.Dp,
                                                   (int)o.Kp, (int)p.Dq, o.xs, o.rex, flag);
  }
  CALS_CUDA_TRY(cudaGetLastError());
  o.flag = flag;
  if (validate) {  // once per tensor and view
    bool keep = true;
    const int rc = ozaki_check(t, key, o, stream, &keep);
    if (rc || !keep) return rc;
  }
  {
    const uint64_t dims[4] = {(uint64_t)o.Kp, (uint64_t)p.M, (uint64_t)p.Dq, (uint64_t)kSlices};
    const uint64_t strides[3] = {(uint64_t)o.Kp, (uint64_t)(p.M * o.Kp),
                                 (uint64_t)(p.Dq * p.M * o.Kp)};
    const uint32_t box[4] = {KSTEP, BNM, 1, kSlices};
    int rc = encode_map_u8(&o.map, o.xs, 4, dims, strides, box);
    if (rc) return rc;
    const MTiling mt = m_tiling(p);
    if (mt.rem_rows) {  // packed remainder tiles: rows M-r.., rem_slabs slabs, one slice
      const uint32_t rbox[4] = {KSTEP, (uint32_t)mt.rem_rows, (uint32_t)mt.rem_slabs, 1};
      rc = encode_map_u8(&o.rmap, o.xs, 4, dims, strides, rbox);
      if (rc) return rc;
    } else {
      o.rmap = o.map;
    }
  }
  std::lock_guard<std::mutex> lk(t.mu);
  if (t.oz.count(key)) {  // another thread raced us: keep theirs
    cudaFreeAsync(o.xs, stream);
    cudaFreeAsync(o.rex, stream);
    if (o.flag) cudaFreeAsync(o.flag, stream);
    return kOk;
  }
  t.oz.emplace(key, o);
  return kOk;
}

bool ozaki_ready(Tensor& t, const ModePlan& p, int key) {
  if (!ozaki_eligible(p)) return false;
  std::lock_guard<std::mutex> lk(t.mu);
  auto it = t.oz.find(key);
  return it != t.oz.end() && !it->second.flag && it->second.M == p.M && it->second.Dq == p.Dq &&
         it->second.Dp == p.Dp;
}

OzLoLayout ozaki_lo_layout(const ModePlan& p, long long lrows, long long cap, void* oz_ws) {
  OzLoLayout l;
  const long long cap_pad = (cap + BMC - 1) / BMC * BMC;
  l.Kp = (int)kp_of(p.Dp);
  l.Dp = (int)std::min<long long>(lrows, p.Dp);
  l.slice_stride = cap_pad * l.Kp;
  l.ls = reinterpret_cast<uint8_t*>(oz_ws);
  l.cex = reinterpret_cast<int*>(
      (reinterpret_cast<uintptr_t>(l.ls + size_t(kSlices) * cap_pad * l.Kp) + 255) &
      ~uintptr_t(255));
  l.queue = l.cex + cap_pad;  // inside the cap_pad * 8 bytes reserved after the slices
  return l;
}

void ozaki_release(Tensor& t) {
  for (auto& kv : t.oz) {
    cudaFreeAsync(kv.second.xs, 0);
    cudaFreeAsync(kv.second.rex, 0);
    if (kv.second.flag) cudaFreeAsync(kv.second.flag, 0);
  }
  t.oz.clear();
}

int launch_contraction_ozaki(Tensor& t, const ModePlan& p, int key, const double* lo,
                             long long lrows, long long lo_ld, const double* hi, long long hi_ld,
                             int width, const int* width_ptr, long long cap, double* out,
                             long long ldo, double* part, void* oz_ws, size_t oz_ws_bytes,
                             cudaStream_t stream, double* side, long long side_ld,
                             long long side_qstride, bool lo_sliced, const int* lo_stale,
                             SplitDefer* defer) {
  OzSlices o;
  {
    std::lock_guard<std::mutex> lk(t.mu);
    auto it = t.oz.find(key);
    if (it == t.oz.end() || it->second.flag) return kErrUnsupported;  // absent / unchecked
    o = it->second;
  }
  CALS_CHECK(o.M == p.M && o.Dq == p.Dq && o.Dp == p.Dp, kErrInvalid, "Ozaki slices / plan mismatch");
  CALS_CHECK(oz_ws && oz_ws_bytes >= ozaki_ws_bytes(p, cap), kErrInvalid,
             "Ozaki workspace too small");
  CALS_CHECK(p.S == 1 || part != nullptr, kErrInvalid, "split-K needs a partial buffer");
  const long long cap_pad = (cap + BMC - 1) / BMC * BMC;
  const OzLoLayout lay = ozaki_lo_layout(p, lrows, cap, oz_ws);
  uint8_t* ls = lay.ls;
  int* cex = lay.cex;
  int* queue = lay.queue;
  const int sms = sm_count(t.device);

  // the one-block-per-column-block kernel wins when there are enough column
  // blocks to fill the GPU (c2: 66 -> 10.6 vs 12.7 us); narrow pools (c3's
  // 10) keep the p-chunked grid (9.0 vs 11.4 us)
  if (lo_sliced) {
    // the kernel that produced Lo also wrote its slices, exponents and the
    // zeroed unit counter (ozaki_lo_layout)
  } else if (o.Kp <= kColsAllMaxKp && (cap + 31) / 32 >= 32) {
    const size_t smem = size_t(o.Kp) * 33 * 8;
    static std::once_flag once;
    static cudaError_t attr = cudaSuccess;
    std::call_once(once, [] {
      attr = cudaFuncSetAttribute(oz_slice_cols_all_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kColsAllMaxKp * 33 * 8);
    });
    CALS_CUDA_TRY(attr);
    CALS_CUDA_TRY(launch_dep(oz_slice_cols_all_kernel, dim3((unsigned)((cap + 31) / 32)), dim3(256),
                             smem, stream, lo, lo_ld, (int)std::min<long long>(lrows, p.Dp),
                             (int)o.Kp, width_ptr, width, (long long)cap_pad, ls, cex, queue,
                             lo_stale));
  } else {
    CALS_CUDA_TRY(launch_dep(oz_slice_cols_kernel,
                             dim3((unsigned)((cap + 31) / 32), (unsigned)(o.Kp / 32)), dim3(256), 0,
                             stream, lo, lo_ld, (int)std::min<long long>(lrows, p.Dp), (int)o.Kp,
                             width_ptr, width, (long long)cap_pad, ls, cex, queue, lo_stale));
  }
  CALS_CUDA_TRY(cudaGetLastError());

  CUtensorMap mapL;
  {
    const uint64_t dims[3] = {(uint64_t)o.Kp, (uint64_t)cap_pad, (uint64_t)kSlices};
    const uint64_t strides[2] = {(uint64_t)o.Kp, (uint64_t)(cap_pad * o.Kp)};
    const uint32_t box[3] = {KSTEP, BMC, kSlices};
    int rc = encode_map_u8(&mapL, ls, 3, dims, strides, box);
    if (rc) return rc;
  }
  Args a{};
  a.M = (int)p.M;
  a.KS = (int)(o.Kp / KSTEP);
  a.Dq = (int)p.Dq;
  a.S = p.S;
  a.width = width;
  a.width_ptr = width_ptr;
  a.hi = hi;
  a.ldh = hi_ld;
  a.rex = o.rex;
  a.cex = cex;
  a.out = p.S > 1 ? part : out;
  a.ldo = p.S > 1 ? lo_ld : ldo;
  a.part_stride = (long long)p.M * lo_ld;
  a.side = side;
  a.ld_side = side_ld;
  a.side_qstride = side_qstride;
  const MTiling mt = m_tiling(p);
  a.tm_full = mt.tm_full;
  a.rem_rows = mt.rem_rows;
  a.rem_slabs = mt.rem_slabs;
  a.queue = queue;
#ifdef CALS_OZ_PROFILE
  // profiling builds: per-CTA cycle counters of the previous launch on stderr
  static unsigned long long* prof = nullptr;
  if (!prof) cudaMalloc(&prof, 148 * 12 * 8);
  a.prof = prof;
  {
    static int calls = 0;
    if (calls++ > 0) {
      unsigned long long h[148 * 12];
      cudaMemcpy(h, prof, sizeof(h), cudaMemcpyDeviceToHost);
      unsigned long long mx = 0, sf = 0, st = 0, ns = 0;
      int wi = 0;
      for (int i = 0; i < 148; ++i) {
        if (h[i * 4] > mx) { mx = h[i * 4]; sf = h[i * 4 + 1]; st = h[i * 4 + 2]; ns = h[i * 4 + 3]; wi = i; }
      }
      for (int k = 0; k < 2; ++k) {
        const unsigned long long* e = h + 148 * 4 + (wi * 2 + k) * 4;
        fprintf(stderr, "[ozprof]   epilogue warp %d: total %llu, wait_tfull %llu, load+release %llu, final %llu\n",
                k ? 5 : 2, e[0], e[1], e[2], e[3]);
      }
      fprintf(stderr, "[ozprof] slowest CTA: total %llu clk, wait_full %llu, wait_tempty %llu, slabs %llu\n",
              mx, sf, st, ns);
    }
  }
#else
  a.prof = nullptr;
#endif

  static std::once_flag attr_once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(attr_once, [] {
    attr_err = cudaFuncSetAttribute(mttkrp_ozaki_kernel<false>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
    if (attr_err == cudaSuccess)
      attr_err = cudaFuncSetAttribute(mttkrp_ozaki_kernel<true>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
  });
  CALS_CUDA_TRY(attr_err);
  const long long units =
      ((cap + BMC - 1) / BMC) * (mt.tm_full + (mt.rem_rows ? 1 : 0)) * (long long)p.S;
  dim3 grid((unsigned)std::max<long long>(1, std::min<long long>(units, sms)));
  if (side)
    CALS_CUDA_TRY(launch_dep(mttkrp_ozaki_kernel<true>, grid, dim3(kThreads), kSmemBytes, stream,
                             o.map, mapL, o.rmap, a));
  else
    CALS_CUDA_TRY(launch_dep(mttkrp_ozaki_kernel<false>, grid, dim3(kThreads), kSmemBytes, stream,
                             o.map, mapL, o.rmap, a));
  CALS_CUDA_TRY(cudaGetLastError());
  if (defer && split_deferrable(p.S, p.M, lo_ld) &&
      !defer->overlaps(part, size_t(p.S) * size_t(a.part_stride) * 8)) {
    *defer = SplitDefer{part, a.part_stride, lo_ld, p.S};
  } else if (p.S > 1) {
    const long long pairs = p.M * ((cap + 1) / 2);
    const int blocks =
        (int)std::max<long long>(1, std::min<long long>(sms * 8, (pairs + 255) / 256));
    CALS_CUDA_TRY(launch_dep(split_reduce_kernel, dim3(blocks), dim3(256), 0, stream,
                             (const double*)part, (long long)a.part_stride, p.S, (int)p.M,
                             (long long)lo_ld, width_ptr, width, out, (long long)ldo));
    CALS_CUDA_TRY(cudaGetLastError());
  }
  return kOk;
}

}  // namespace cals
