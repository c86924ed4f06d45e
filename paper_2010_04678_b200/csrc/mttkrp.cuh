// Fused multi-model MTTKRP for sm_100a on FP64 tensor cores (DMMA.8x8x4).
//
// Replaces the reference's numpy/OpenBLAS MTTKRP variants
// (pkg/src/cals/mttkrp.py:157-256: FIRST = KRP materialise + dgemm,
// MIDDLE = per-slab dgemm + row scaling, LAST = KRP materialise + dgemm).
//
// Every mode-n MTTKRP of a dense tensor (mode-0 fastest) is viewed as a
// contiguous 3-D array (D0, D1, D2) in which one dimension is the output row
// index m, one is the "p" index contracted on the tensor cores against the
// factor Lo[p, c], and one is the "q" index whose factor Hi[q, c] scales the
// per-slab product column-wise:
//
//     M[m, c] = sum_q Hi[q, c] * ( sum_p X[m, p, q] * Lo[p, c] ).
//
// This is the Khatri-Rao product applied in factored form: no KRP panel is
// ever formed (the probe in profiles/r01_fp64_peak_probe.txt shows DMUL
// interleaved with DMMA costs ~25-50% of DMMA throughput on B200), the inner
// contraction is a plain DMMA GEMM with both operands streamed by TMA, and the
// KRP costs one DFMA per accumulator element per q-slab.  Roles:
//   FIRST  (mode 0):   view (m, p, q),   A tile smem [k][m]  (m contiguous)
//   MIDDLE (interior): view (p, m, q),   A tile smem [m][k]  (k contiguous)
//   LAST   (mode N-1): view (p, q, m),   A tile smem [m][k]
// so the middle mode needs no transposed copy of the tensor.
//
// Tall-K: the q range is split S ways (S depends only on the tensor shape,
// never on the active width), each split writes a partial slab and a
// fixed-order reduction sums them -> results are deterministic and bitwise
// independent of a model's column position and of the other models present.
#pragma once

#include "common.cuh"

namespace cals {

// FIRST_QP: view (m, q, p) -- mode 0 with the slab index on dim 1 and the
// contracted index on dim 2; its per-slab products are the dimension-tree
// partial Y[i, j, :] = sum_k X[i,j,k] A2[k, :] (see `side` below).
enum Role : int { kRoleFirst = 0, kRoleMiddle = 1, kRoleLast = 2, kRoleFirstQP = 3 };

constexpr int kBK = 16;   // p-tile (DMMA k extent per pipeline stage)
constexpr int kPad = 4;   // extra inner-dimension elements per smem row: pitch = 4 mod 16
                          // doubles makes every DMMA fragment load bank-conflict free

struct MttkrpArgs {
  int role;
  int M;               // output rows
  int Dp;              // contracted (tensor-core k) extent
  int Dq;              // scaled-slab extent
  int S;               // q splits (>= 1)
  int width;           // active width when width_ptr == nullptr
  const int* width_ptr;
  const double* hi;    // [Dq][ldh]
  long long ldh;
  double* out;         // S == 1: [M][ldo]; S > 1: partials [S][M][ldo]
  long long ldo;
  long long part_stride;
  // optional side output of every per-slab product (before the Hi scaling):
  // side[(m + side_qstride * q) * ld_side + c]  -- the dimension-tree partial
  double* side;
  long long ld_side;
  long long side_qstride;
};

template <int MI, int NI, int WM, int WN>
struct TileCfg {
  static constexpr int BM = 8 * MI * WM;
  static constexpr int BN = 8 * NI * WN;
  static constexpr int kConsumerWarps = WM * WN;
  static constexpr int kThreads = 32 * (kConsumerWarps + 1);
  static constexpr int A_K_ELEMS = BM * (kBK + kPad);   // [m][k] layout
  static constexpr int A_M_ELEMS = kBK * (BM + kPad);   // [k][m] layout
  static constexpr int A_ELEMS = A_K_ELEMS > A_M_ELEMS ? A_K_ELEMS : A_M_ELEMS;
  static constexpr int B_ELEMS = kBK * (BN + kPad);
  static constexpr int STAGES = 4;
  static constexpr size_t kStageBytes = size_t(A_ELEMS + B_ELEMS) * 8;
  static constexpr size_t kAccBytes = size_t(kConsumerWarps) * 32 * MI * NI * 2 * 8;
  static constexpr size_t kBarBytes = 2 * STAGES * 8;
  static constexpr size_t kSmemBytes = STAGES * kStageBytes + kBarBytes + kAccBytes + 128;
};

// p-tile `pt` loads the kBK-wide box at p0 and consumes its k4 steps
// [ks_lo, ks_hi).  A ragged last tile is shifted left onto a multiple of 4 and
// its already-consumed leading steps skipped, so no DMMA is spent on padding
// beyond the last k4 group (Dp = 200 -> exactly 50 k4 steps).
__device__ __forceinline__ void ptile(int pt, int Dp, int& p0, int& ks_lo, int& ks_hi) {
  p0 = pt * kBK;
  ks_lo = 0;
  const int rem = Dp - p0;
  if (rem < kBK && pt > 0) {
    const int j = (kBK - rem) >> 2;
    p0 -= 4 * j;
    ks_lo = j;
  }
  ks_hi = min(kBK / 4, (Dp - p0 + 3) >> 2);
}

__device__ __forceinline__ void unit_decode(int u, int tm, int tn, int& tile_m, int& tile_n,
                                            int& s) {
  tile_n = u % tn;
  int t = u / tn;
  tile_m = t % tm;
  s = t / tm;
}

template <int MI, int NI, int WM, int WN, bool KC>
// 2 CTAs x 5 warps per SM: some SMSP holds 3 warps, and each SMSP's register
// file is 16K 32-bit registers -> at most 168 registers per thread.
__global__ void __launch_bounds__(TileCfg<MI, NI, WM, WN>::kThreads, 2)
    mttkrp_dmma_kernel(const __grid_constant__ CUtensorMap tmA,
                       const __grid_constant__ CUtensorMap tmB, const MttkrpArgs args) {
  using C = TileCfg<MI, NI, WM, WN>;
  constexpr int BM = C::BM, BN = C::BN, STAGES = C::STAGES;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* smem = reinterpret_cast<double*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + STAGES * C::kStageBytes);
  uint64_t* empty = full + STAGES;

  griddep_wait();  // launched with PDL (launch_dep): predecessors complete
  const int W = args.width_ptr ? *args.width_ptr : args.width;
  if (W <= 0) return;
  const int tm = (args.M + BM - 1) / BM;
  const int tn = (W + BN - 1) / BN;
  const int units = tm * tn * args.S;
  const int np = (args.Dp + kBK - 1) / kBK;
  const uint32_t a_bytes = uint32_t(KC ? C::A_K_ELEMS : C::A_M_ELEMS) * 8u;
  const uint32_t stage_tx = a_bytes + uint32_t(C::B_ELEMS) * 8u;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], C::kConsumerWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == C::kConsumerWarps) {
    // ===================== TMA producer (one elected lane) ==================
    if (lane == 0) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmB);
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        int tile_m, tile_n, s;
        unit_decode(u, tm, tn, tile_m, tile_n, s);
        const int qb = int((long long)s * args.Dq / args.S);
        const int qe = int((long long)(s + 1) * args.Dq / args.S);
        const int m0 = tile_m * BM, c0 = tile_n * BN;
        for (int q = qb; q < qe; ++q) {
          for (int pt = 0; pt < np; ++pt) {
            mbar_wait(&empty[stage], phase ^ 1u);
            double* sa = smem + size_t(stage) * (C::A_ELEMS + C::B_ELEMS);
            double* sb = sa + C::A_ELEMS;
            mbar_arrive_expect_tx(&full[stage], stage_tx);
            int p0, ks_lo, ks_hi;
            ptile(pt, args.Dp, p0, ks_lo, ks_hi);
            if (args.role == kRoleFirst)
              tma_load_3d(sa, &tmA, &full[stage], m0, p0, q);
            else if (args.role == kRoleMiddle)
              tma_load_3d(sa, &tmA, &full[stage], p0, m0, q);
            else if (args.role == kRoleLast)
              tma_load_3d(sa, &tmA, &full[stage], p0, q, m0);
            else
              tma_load_3d(sa, &tmA, &full[stage], m0, q, p0);
            tma_load_2d(sb, &tmB, &full[stage], c0, p0);
            if (++stage == STAGES) { stage = 0; phase ^= 1u; }
          }
        }
      }
    }
    return;
  }

  // ======================= DMMA consumers =====================================
  const int wm = warp / WN, wn = warp % WN;
  double* accs = reinterpret_cast<double*>(smem_raw + STAGES * C::kStageBytes + C::kBarBytes) +
                 size_t(warp) * (MI * NI * 2) * 32 + lane;
  const int r = lane >> 2, kq = lane & 3;
  int stage = 0;
  uint32_t phase = 0;
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    int tile_m, tile_n, s;
    unit_decode(u, tm, tn, tile_m, tile_n, s);
    const int qb = int((long long)s * args.Dq / args.S);
    const int qe = int((long long)(s + 1) * args.Dq / args.S);
    const int m0 = tile_m * BM, c0 = tile_n * BN;
    const int cw = c0 + wn * 8 * NI + 2 * kq;  // this lane's first column

    // The cross-slab accumulator lives in shared memory (this lane's column
    // of a per-warp [element][lane] block): it is touched once per q-slab,
    // and keeping it out of registers leaves the whole register budget to
    // the DMMA tile and its pipelined fragments.
#pragma unroll
    for (int e = 0; e < MI * NI * 2; ++e) accs[e * 32] = 0.0;

    for (int q = qb; q < qe; ++q) {
      double t[MI][NI][2];
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) t[i][j][0] = t[i][j][1] = 0.0;

      auto run_stage = [&](int pt) {
        mbar_wait(&full[stage], phase);
        const double* sa = smem + size_t(stage) * (C::A_ELEMS + C::B_ELEMS);
        const double* sb = sa + C::A_ELEMS;
        int p0, ks_lo, ks_hi;
        ptile(pt, args.Dp, p0, ks_lo, ks_hi);
        auto kstep = [&](int ks) {
          const int k = 4 * ks + kq;
          double a[MI], b[NI];
          if constexpr (KC) {
#pragma unroll
            for (int i = 0; i < MI; ++i)
              a[i] = sa[(wm * 8 * MI + 8 * i + r) * (kBK + kPad) + k];
          } else {
#pragma unroll
            for (int i = 0; i < MI; ++i) a[i] = sa[k * (BM + kPad) + wm * 8 * MI + 8 * i + r];
          }
#pragma unroll
          for (int j = 0; j < NI; ++j) b[j] = sb[k * (BN + kPad) + wn * 8 * NI + 8 * j + r];
#pragma unroll
          for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int j = 0; j < NI; ++j) dmma_8x8x4(t[i][j][0], t[i][j][1], a[i], b[j]);
        };
        if (ks_lo == 0 && ks_hi == kBK / 4) {
          // full tile: branch-free, so fragment loads of step ks+1 overlap the
          // DMMAs of step ks
#pragma unroll
          for (int ks = 0; ks < kBK / 4; ++ks) kstep(ks);
        } else {
#pragma unroll 1
          for (int ks = ks_lo; ks < ks_hi; ++ks) kstep(ks);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1u; }
      };
      for (int pt = 0; pt < np - 1; ++pt) run_stage(pt);
      // Hi[q] is only live across the last p-tile (its latency hides behind
      // that tile's DMMAs) -- keeps the main loop within the register budget
      double hi[NI][2];
      const double* hrow = args.hi + (long long)q * args.ldh;
#pragma unroll
      for (int j = 0; j < NI; ++j) {
        const int c = cw + 8 * j;
        hi[j][0] = c < W ? __ldg(hrow + c) : 0.0;
        hi[j][1] = c + 1 < W ? __ldg(hrow + c + 1) : 0.0;
      }
      run_stage(np - 1);
      if (args.side) {
        // dimension-tree partial: the unscaled slab product, written once
#pragma unroll
        for (int i = 0; i < MI; ++i) {
          const int m = m0 + wm * 8 * MI + 8 * i + r;
          if (m >= args.M) continue;
          double* srow = args.side + ((long long)m + args.side_qstride * q) * args.ld_side;
#pragma unroll
          for (int j = 0; j < NI; ++j) {
            const int c = cw + 8 * j;
            if (c + 1 < W)
              __stcg(reinterpret_cast<double2*>(srow + c), make_double2(t[i][j][0], t[i][j][1]));
            else if (c < W)
              __stcg(srow + c, t[i][j][0]);
          }
        }
      }
      // Khatri-Rao factor of the q-slab: one DFMA per accumulator element.
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) {
          double* a2 = accs + ((i * NI + j) * 2) * 32;
          a2[0] = fma(t[i][j][0], hi[j][0], a2[0]);
          a2[32] = fma(t[i][j][1], hi[j][1], a2[32]);
        }
    }

    double* out = args.out + (args.S > 1 ? (long long)s * args.part_stride : 0LL);
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int m = m0 + wm * 8 * MI + 8 * i + r;
      if (m >= args.M) continue;
      double* orow = out + (long long)m * args.ldo;
#pragma unroll
      for (int j = 0; j < NI; ++j) {
        const int c = cw + 8 * j;
        const double* a2 = accs + ((i * NI + j) * 2) * 32;
        if (c + 1 < W) {
          *reinterpret_cast<double2*>(orow + c) = make_double2(a2[0], a2[32]);
        } else if (c < W) {
          orow[c] = a2[0];
        }
      }
    }
  }
}

// out[m][c] = sum_{s ascending} part[s][m][c]  (deterministic split reduction)
__global__ void split_reduce_kernel(const double* __restrict__ part, long long part_stride,
                                    int S, int M, long long ldp, const int* width_ptr, int width,
                                    double* __restrict__ out, long long ldo);

}  // namespace cals
