// FP64-accurate fused MTTKRP on the sm_100a INT8 tensor cores (tcgen05.mma
// kind::i8, accumulators in TMEM, operands staged by TMA) -- Ozaki-scheme
// slicing of both operands.
//
// Same contraction as mttkrp.cuh (pkg/src/cals/mttkrp.py:157-256 restated in
// factored form):
//
//     M[m, c] = sum_q Hi[q, c] * P_q[m, c],   P_q[m, c] = sum_p X[m, p, q] * Lo[p, c]
//
// but the slab product P_q is computed exactly from integer slices instead of
// on the (warp-level, ~37 TFLOP/s) FP64 DMMA pipe.  Every row (q, m) of the
// tensor view and every column c of Lo is scaled by a power of two 2^e with
// max|v| < 2^e and cut into 7 slices
//
//     v = 2^e * ( s1 2^-7 + s2 2^-15 + s3 2^-23 + ... + s7 2^-55 + r ),
//     s1 = floor(v 2^(7-e)) in [-128, 127] (int8),  s2..s7 in [0, 255] (uint8),
//     0 <= r < 2^-55,
//
// all exact in FP64.  The 28 slice products with i + j <= 8 are accumulated
// exactly in int32 TMEM accumulators, one per "group" g = i + j (the groups
// are 2^8 apart in weight), and the epilogue recombines them by Horner in
// 64-bit integers:  P = 2^(ex + el - 62) * sum_g A_g 2^(8 (8 - g)).  Truncation error per
// term <= ~2^-50.6 * 2^(ex + el) -- the same order as the DGEMM it replaces
// (K * 2^-53 * sum |x||lo|), see DESIGN.md section 4.1b.
//
// The X slices depend only on the (immutable) tensor and are built once per
// tensor and view; the Lo slices are rebuilt per call (a few MB).
//
// CTA tile: 128 Lo columns c (the MMA M dimension = TMEM lanes) x 64 tensor
// rows m (MMA N); K steps of 32 p.  Warp 0 = TMA producer, warp 1 = MMA
// issuer (one thread), warps 2..9 = epilogue (TMEM -> registers -> FP64).
// TMEM: 8 rotating buffers x 64 columns for the 7 groups.  Each group's accumulator is
// committed to its own mbarrier as soon as its last product of the slab is
// issued and released by the epilogue as soon as it has been read, so the
// epilogue of slab q overlaps the tail of slab q and the head of slab q+1.
//
// Determinism / position independence: a column's result depends only on its
// own Lo column, the shape-only X slicing and a fixed operation order (Horner
// over groups, ascending q inside a split, fixed-order split reduction).
#pragma once

#include "common.cuh"
#include "tcgen05.cuh"

namespace cals {
namespace oz {

constexpr int kSlices = 7;
// Tensor rows whose median nonzero magnitude is below 2^-kRangeBits of the row
// maximum keep < 55 - kRangeBits bits in most entries: such views stay on DMMA.
constexpr int kRangeBits = 20;
constexpr int kGroups = 7;   // g = i + j in [2, 8]
constexpr int BMC = 128;     // c per tile (MMA M, TMEM lanes)
constexpr int BNM = 64;      // m per tile (MMA N)
constexpr int KSTEP = 32;    // int8 K per tcgen05.mma
constexpr int STAGES = 3;
constexpr int kLoTileBytes = BMC * KSTEP;              // 4096 per slice
constexpr int kXTileBytes = BNM * KSTEP;               // 2048 per slice
constexpr int kLoStageBytes = kSlices * kLoTileBytes;  // 28672
constexpr int kXStageBytes = kSlices * kXTileBytes;    // 14336
constexpr int kStageBytes = kLoStageBytes + kXStageBytes;
constexpr int kEpiWarps = 8;
constexpr int kThreads = 32 * (2 + kEpiWarps);
constexpr int kTmemCols = 512;
// 8 accumulator buffers of 64 columns rotate over the 7 groups: group g of
// the s-th slab uses buffer (7 s + g) mod 8, so the next slab's group g
// overwrites the buffer of this slab's group g - 1 (drained one group
// earlier) -- one group of slack between the epilogue and the MMA warp.
constexpr int kTmemBufs = 8;
#ifdef CALS_OZ_PROFILE
constexpr bool kProfile = true;
#else
constexpr bool kProfile = false;
#endif
__device__ __forceinline__ long long prof_clock() { return kProfile ? clock64() : 0; }
// cross-slab FP64 accumulator of the epilogue: [32 rows m][256 epilogue threads]
constexpr size_t kAccBytes = size_t(32) * 32 * kEpiWarps * 8;
constexpr size_t kSmemBytes =
    size_t(STAGES) * kStageBytes + kAccBytes + 1024 /*align*/ + 512 /*barriers, unit ring*/;
// work units are handed out at run time (atomic counter, largest units
// first): the producer warp claims the next unit and passes it to the MMA and
// epilogue warps through a small ring in shared memory
constexpr int kUnitRing = 4;

struct Args {
  int M;        // tensor rows of the view (output rows)
  int KS;       // K steps of 32 (Kp / 32)
  int Dq;       // slabs
  int S;        // q splits
  int width;    // active width if width_ptr == nullptr
  const int* width_ptr;
  const double* hi;  // [Dq][ldh]
  long long ldh;
  const int* rex;     // [Dq][M] row scale exponents ex of the X slices
  const int* cex;     // [>= W] column scale exponents el of the Lo slices
  double* out;       // S == 1: [M][ldo]; else partials [S][M][ldo]
  long long ldo;
  long long part_stride;
  double* side;      // optional per-slab products side[(m + side_qstride q) * ld_side + c]
  long long ld_side;
  long long side_qstride;
  // m tiling: tm_full tiles of 64 rows; if rem_rows > 0 the last M % 64 rows
  // of every slab of a q-split are packed into ONE extra 64-row tile
  // (rem_rows x rem_slabs rows, slab-major), so a 200-row mode costs 3 + 1/6
  // instead of 4 tile passes per slab.
  int tm_full;
  int rem_rows;
  int rem_slabs;
  // unit counter, zeroed by the Lo slicing kernel before every launch
  int* queue;
  // CALS_OZ_PROFILE builds only: per-CTA cycle counters (MMA waits, epilogue
  // phases) -- see tools/oz_time.py
  unsigned long long* prof;
};

// ------------------------------------------------------------ instruction --
// kind::i8 instruction descriptor: S32 accumulate, K-major A and B, M = 128, N = 64
__host__ __device__ constexpr uint32_t idesc_i8(int a_signed, int b_signed) {
  return (2u << 4) | ((uint32_t)a_signed << 7) | ((uint32_t)b_signed << 10) |
         ((uint32_t)(BNM >> 3) << 17) | ((uint32_t)(BMC >> 4) << 24);
}
// ------------------------------------------------------------------ slicing --
// v in (-2^e, 2^e): 7 slices, s1 signed, s2..s7 unsigned (see header).  The
// slices are the base-256 digits of Y = floor(v 2^(55-e)) (|Y| < 2^55): the
// scaling is by a power of two and floor is exact, so one multiply and one
// conversion give all seven exactly (the top digit as a signed byte).
__device__ __forceinline__ void slice7(double v, int e, uint8_t (&s)[kSlices]) {
  const int k = 55 - e;
  const double t = (k >= -1022 && k <= 1023) ? v * __hiloint2double((k + 1023) << 20, 0)
                                             : ldexp(v, k);
  const long long y = __double2ll_rd(t);
  s[0] = (uint8_t)(y >> 48);
#pragma unroll
  for (int i = 1; i < kSlices; ++i) s[i] = (uint8_t)(y >> (48 - 8 * i));
}
// Lo columns holding a NaN or Inf get this scale exponent: their slices are
// zero and the epilogue emits NaN for them (as the FP64 contraction would).
// A tensor with a non-finite entry is left to the DMMA kernel.
constexpr int kNonFinite = 1 << 20;
__device__ __forceinline__ double abs_or_inf(double v) {
  const double a = fabs(v);
  return a <= 1.7976931348623157e308 ? a : __longlong_as_double(0x7ff0000000000000LL);
}
__device__ __forceinline__ int scale_exp_checked(double amax);

// smallest e with max|v| < 2^e (0 for an all-zero vector)
__device__ __forceinline__ int scale_exp(double amax) { return amax > 0.0 ? ilogb(amax) + 1 : 0; }
__device__ __forceinline__ int scale_exp_checked(double amax) {
  return amax <= 1.7976931348623157e308 ? scale_exp(amax) : kNonFinite;
}

// Work unit u (c fastest): a full 64-row m-tile over the slabs of one q-split,
// or the split's packed remainder tile (one pass, rem_rows x slabs rows).
struct Unit {
  int tc, s, qb, qe, m0;
  bool rem;
};
__device__ __forceinline__ Unit unit_decode(int u, int tn, const Args& a) {
  Unit U;
  U.tc = u % tn;
  const int t = u / tn;
  const int full = a.tm_full * a.S;
  U.rem = t >= full;
  U.s = U.rem ? t - full : t / a.tm_full;
  U.m0 = U.rem ? a.M - a.rem_rows : (t % a.tm_full) * BNM;
  U.qb = int((long long)U.s * a.Dq / a.S);
  U.qe = int((long long)(U.s + 1) * a.Dq / a.S);
  return U;
}

// v * 2^k for v = (double) of an integer (0 or |v| in [1, 2^62)) and an
// exponent k keeping the result normal: integer add on the exponent field
__device__ __forceinline__ double exp_add(double v, int k) {
  const int hi = __double2hiint(v);
  return (hi & 0x7ff00000) ? __hiloint2double(hi + (k << 20), __double2loint(v)) : 0.0;
}

// 2^e as a double: exponent-field construction in the normal range, ldexp
// (subnormal / zero / inf) outside it
__device__ __forceinline__ double pow2(int e) {
  if (e < -1022 || e > 1023) return ldexp(1.0, e);
  return __hiloint2double((e + 1023) << 20, 0);
}

// Epilogue: drain one pass's 7 group accumulators (each TMEM buffer released
// to the MMA warp as soon as it is in registers) and recombine them in 64-bit
// integers into P (the double of Q ~ P' / 2^12, see the kernel comment).
__device__ __forceinline__ void drain_pass(uint64_t* tfull, uint64_t* tempty, uint32_t slab,
                                           uint32_t trow, int lane, double (&P)[32],
                                           long long& ew_wait, long long& ew_load) {
  uint32_t v[32];
  long long Qv[32];
#pragma unroll
  for (int g = 0; g < kGroups; ++g) {
    const long long e0 = prof_clock();
    const uint32_t L = 7u * slab + g, buf = L & 7u;
    mbar_wait(&tfull[buf], (L >> 3) & 1u);
    tc_fence_after();
    const long long e1 = prof_clock();
    ew_wait += e1 - e0;
    tmem_ld32(trow + buf * BNM, v);
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&tempty[buf]);  // TMEM buffer free for its next use
    ew_load += prof_clock() - e1;
    if (g == 0) {
#pragma unroll
      for (int j = 0; j < 32; ++j) Qv[j] = (long long)(int)v[j];
    } else if (g <= 4) {
#pragma unroll
      for (int j = 0; j < 32; ++j) Qv[j] = Qv[j] * 256 + (long long)(int)v[j];
    } else if (g == 5) {
#pragma unroll
      for (int j = 0; j < 32; ++j) Qv[j] = Qv[j] * 16 + (long long)((int)v[j] >> 4);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) P[j] = (double)(Qv[j] + (long long)((int)v[j] >> 12));
    }
  }
}

// Consumer side of the unit ring (MMA warp, epilogue warps): wait for the
// producer's claim, read it, release the slot.
__device__ __forceinline__ int next_unit(uint64_t* ufull, uint64_t* uempty, const int* uring,
                                         int& uslot, uint32_t& uphase, int lane) {
  mbar_wait(&ufull[uslot], uphase);
  const int u = uring[uslot];
  __syncwarp();
  if (lane == 0) mbar_arrive(&uempty[uslot]);
  if (++uslot == kUnitRing) { uslot = 0; uphase ^= 1u; }
  return u;
}

// ------------------------------------------------------------- main kernel --
// kSide: the launch writes the per-slab products (dimension-tree partial);
// a separate instantiation keeps the side-output code out of the other
// launches (measured 7 % of the kernel even when skipped at run time).
template <bool kSide>
__global__ void __launch_bounds__(kThreads, 1)
    mttkrp_ozaki_kernel(const __grid_constant__ CUtensorMap tmX,
                        const __grid_constant__ CUtensorMap tmL,
                        const __grid_constant__ CUtensorMap tmR, const Args args) {
  // dynamic shared memory starts at the CTA window base (no static smem in
  // this kernel): 1024-byte aligned, as the 32-byte swizzle atoms need.  No
  // pointer arithmetic through integers, so accesses stay LDS/STS.
  extern __shared__ __align__(1024) unsigned char smem[];
  double* acc_s = reinterpret_cast<double*>(smem + STAGES * kStageBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kStageBytes + kAccBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + kTmemBufs;
  uint64_t* ufull = tempty + kTmemBufs;
  uint64_t* uempty = ufull + kUnitRing;
  int* uring = reinterpret_cast<int*>(uempty + kUnitRing);
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(uring + kUnitRing);

  if ((smem_u32(smem) & 1023u) != 0) __trap();
  griddep_wait();  // launched with PDL (launch_dep): predecessors complete
  const int W = args.width_ptr ? *args.width_ptr : args.width;
  if (W <= 0) return;
  const int tn = (W + BMC - 1) / BMC;
  const int units = tn * (args.tm_full + (args.rem_rows ? 1 : 0)) * args.S;
  if ((int)blockIdx.x >= units) return;
  const int KS = args.KS;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int b = 0; b < kTmemBufs; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kEpiWarps);
    }
    for (int b = 0; b < kUnitRing; ++b) {
      mbar_init(&ufull[b], 1);
      mbar_init(&uempty[b], 1 + kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_base_slot)),
                 "n"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_base_slot;

  if (warp == 0) {
    // ============================ TMA producer =================================
    if (lane == 0) {
      tma_prefetch_desc(&tmX);
      tma_prefetch_desc(&tmL);
      int stage = 0;
      uint32_t phase = 0;
      tma_prefetch_desc(&tmR);
      const uint32_t rem_tx =
          uint32_t(kLoStageBytes + kSlices * KSTEP * args.rem_rows * args.rem_slabs);
      int uslot = 0;
      uint32_t uphase = 0;
      for (;;) {
        // claim the next unit (units are numbered largest first: full tiles,
        // then the one-pass remainder tiles) and publish it to the ring
        mbar_wait(&uempty[uslot], uphase ^ 1u);
        int u = atomicAdd(args.queue, 1);
        if (u >= units) u = -1;
        uring[uslot] = u;
        mbar_arrive(&ufull[uslot]);
        if (++uslot == kUnitRing) { uslot = 0; uphase ^= 1u; }
        if (u < 0) break;
        const Unit U = unit_decode(u, tn, args);
        const int passes = U.rem ? 1 : U.qe - U.qb;
        for (int i = 0; i < passes; ++i) {
          const int q = U.qb + i;
          for (int ks = 0; ks < KS; ++ks) {
            mbar_wait(&empty[stage], phase ^ 1u);
            unsigned char* st = smem + size_t(stage) * kStageBytes;
            if (U.rem) {
              // rows M-r..M-1 of slabs qb.. (rem_slabs of them), one box per
              // slice at the slice's 2048-byte B-tile offset
              mbar_arrive_expect_tx(&full[stage], rem_tx);
              tma_load_3d(st, &tmL, &full[stage], ks * KSTEP, U.tc * BMC, 0);
              for (int j = 0; j < kSlices; ++j)
                tma_load_4d(st + kLoStageBytes + j * kXTileBytes, &tmR, &full[stage], ks * KSTEP,
                            U.m0, U.qb, j);
            } else {
              mbar_arrive_expect_tx(&full[stage], kStageBytes);
              tma_load_3d(st, &tmL, &full[stage], ks * KSTEP, U.tc * BMC, 0);
              tma_load_4d(st + kLoStageBytes, &tmX, &full[stage], ks * KSTEP, U.m0, q, 0);
            }
            if (++stage == STAGES) { stage = 0; phase ^= 1u; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer ===================================
    // The whole warp runs the loop and one elected lane issues.  Interior K
    // steps issue their 28 products from one asm block; the first K step of
    // a slab waits per group for the epilogue to release its accumulator, and
    // the last commits each group as soon as its final product is issued.
    int stage = 0;
    uint32_t phase = 0;
    uint32_t slab = 0;
    const uint64_t sdesc = desc_sw32(smem_u32(smem));
    long long w_full = 0, w_tempty = 0;
    const long long t_start = prof_clock();
    int uslot = 0;
    uint32_t uphase = 0;
    for (;;) {
      const int u = next_unit(ufull, uempty, uring, uslot, uphase, lane);
      if (u < 0) break;
      const Unit U = unit_decode(u, tn, args);
      const int passes = U.rem ? 1 : U.qe - U.qb;
      for (int i = 0; i < passes; ++i, ++slab) {
        // group g of this slab -> buffer (7 slab + g) mod 8, use (7 slab + g) / 8
        const uint32_t L0 = 7u * slab;
        uint32_t d[7];
#pragma unroll
        for (int g = 0; g < kGroups; ++g) d[g] = tmem + ((L0 + g) & 7u) * BNM;
        for (int ks = 0; ks < KS; ++ks) {
          // descriptor start-address field counts 16-byte units
          const uint64_t a0 = sdesc + (uint64_t)((stage * kStageBytes) >> 4);
          const uint64_t b0 = a0 + (uint64_t)(kLoStageBytes >> 4);
          if (ks > 0 && ks < KS - 1) {
            // interior K step: wait, 28 products, release -- one asm block
            issue_kstep_mid(d, a0, b0, smem_u32(&full[stage]), phase, smem_u32(&empty[stage]));
            if (++stage == STAGES) { stage = 0; phase ^= 1u; }
            continue;
          }
          long long t0 = prof_clock();
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          w_full += prof_clock() - t0;
          if (ks > 0) {
            {
              uint32_t bar[7];
#pragma unroll
              for (int g = 0; g < kGroups; ++g) bar[g] = smem_u32(&tfull[(L0 + g) & 7u]);
              issue_kstep_last(d, a0, b0, bar);
            }
          } else if (KS > 1) {
            uint32_t bar[7], par[7];
#pragma unroll
            for (int g = 0; g < kGroups; ++g) {
              const uint32_t buf = (L0 + g) & 7u, use = (L0 + g) >> 3;
              bar[g] = smem_u32(&tempty[buf]);
              par[g] = (use & 1u) ^ 1u;
            }
            issue_kstep_first(d, a0, b0, bar, par);
          } else {
            // a single K step: first and last at once (per-group waits and commits)
#pragma unroll
            for (int g = 0; g < kGroups; ++g) {
              const int sum = g + 2;
              const int i_lo = sum - kSlices > 1 ? sum - kSlices : 1;
              const int i_hi = sum - 1 < kSlices ? sum - 1 : kSlices;
              const uint32_t buf = (L0 + g) & 7u, use = (L0 + g) >> 3;
              if (ks == 0) {
                // the epilogue must have drained this buffer's previous use
                long long t1 = prof_clock();
                mbar_wait(&tempty[buf], (use & 1u) ^ 1u);
                tc_fence_after();
                w_tempty += prof_clock() - t1;
              }
#pragma unroll
              for (int i = i_lo; i <= i_hi; ++i) {
                const int j = sum - i;
                mma_i8_elect(tmem + buf * BNM, a0 + (uint64_t)(((i - 1) * kLoTileBytes) >> 4),
                             b0 + (uint64_t)(((j - 1) * kXTileBytes) >> 4),
                             idesc_i8(i == 1, j == 1), (ks > 0 || i != i_lo) ? 1u : 0u);
              }
              if (ks == KS - 1) tc_commit_elect(&tfull[buf]);
            }
          }
          tc_commit_elect(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1u; }
        }
      }
    }
    if (kProfile && lane == 0) {
      args.prof[blockIdx.x * 4 + 0] = prof_clock() - t_start;
      args.prof[blockIdx.x * 4 + 1] = w_full;
      args.prof[blockIdx.x * 4 + 2] = w_tempty;
      args.prof[blockIdx.x * 4 + 3] = slab;
    }
  } else {
    // ============================ epilogue =====================================
    // The FP64 pipe is shared with the tensor cores: every FP64 instruction
    // issued here waits for, and costs, MMA time, while the integer pipe and
    // the conversion unit (I2F) overlap the MMAs.  So the groups are combined
    // in 64-bit integers,
    //   Q = sum_{g<=4} A_g 2^(8(4-g)) * 16 + (A_5 >> 4) + (A_6 >> 12)  ~ P' / 2^12,
    //   P' = sum_g A_g 2^(8(6-g)),  P_q[m][c] = 2^(ex + el - 50) * Q,
    // (|Q| < 2^62 for K <= 2048; the dropped bits are < 2^-50 of
    // max|x| max|lo|, inside the slicing error), converted once (I2F), and
    // the per-element FP64 work is one DMUL (row scale) + one DFMA (Hi).
    const int quad = warp & 3;             // TMEM lane quadrant this warp may access
    const int half = (warp - 2) >> 2;      // which 32 of the tile's 64 rows m
    const uint32_t trow = tmem + ((uint32_t)(quad * 32) << 16) + half * 32;
    uint32_t slab = 0;
    long long ew_wait = 0, ew_load = 0, ew_final = 0;
    const long long e_start = prof_clock();
    int uslot = 0;
    uint32_t uphase = 0;
    for (;;) {
      const int u = next_unit(ufull, uempty, uring, uslot, uphase, lane);
      if (u < 0) break;
      const Unit U = unit_decode(u, tn, args);
      const int c = U.tc * BMC + quad * 32 + lane;
      const bool cval = c < W;
      const int mb = U.m0 + half * 32;
      const int el = cval ? args.cex[c] : 0;
      const int kside = el - 50;
      const double kNaN = __longlong_as_double(0x7ff8000000000000LL);
      const double cscale = !cval ? 0.0 : (el == kNonFinite ? kNaN : pow2(kside));
      // exponent-add fast path for the side output: |ex| <= 900 and the
      // result exponent field e_P + ex + kside (e_P in [1023, 1085]) in range
      const bool side_fast = __all_sync(0xffffffffu, kside >= -122 && kside <= 61);
      // this thread's accumulator column in shared memory (touched once per
      // slab; keeps the registers for the TMEM values)
      double* acc = acc_s + (threadIdx.x - 64);
      // Drain this pass's 7 group accumulators (each released to the MMA warp
      // as soon as it is in registers) and recombine them into P (see above).
      double P[32];
      if (!U.rem) {
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[j * 32 * kEpiWarps] = 0.0;
        for (int q = U.qb; q < U.qe; ++q, ++slab) {
          const double hc = cval ? __ldg(args.hi + (long long)q * args.ldh + c) * cscale : 0.0;
          // row scales of this warp's 32 rows: one coalesced load, broadcast
          // by shuffles (its latency hides behind the group drain)
          const int rex_lane =
              mb + lane < args.M ? __ldg(args.rex + (long long)q * args.M + mb + lane) : 0;
          drain_pass(tfull, tempty, slab, trow, lane, P, ew_wait, ew_load);
          const long long e2 = prof_clock();
          // Scaling by 2^ex (row) and 2^(ex + el - 50) (side output) is an
          // exponent-field add on the integer pipe: P is the double of an
          // integer (0, or |P| in [1, 2^62)), row exponents are confined to
          // [-900, 900] (ozaki_prepare falls back to DMMA otherwise) and the
          // column term is checked per warp.  One DFMA per element is left.
          if (side_fast) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int m = mb + j;
              const int ex = __shfl_sync(0xffffffffu, rex_lane, j);
              const double y = exp_add(P[j], ex);
              if (kSide && cval && m < args.M)
                __stcg(args.side + ((long long)m + args.side_qstride * q) * args.ld_side + c,
                       exp_add(P[j], ex + kside));
              acc[j * 32 * kEpiWarps] = fma(y, hc, acc[j * 32 * kEpiWarps]);
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int m = mb + j;
              const double y = exp_add(P[j], __shfl_sync(0xffffffffu, rex_lane, j));
              if (kSide && cval && m < args.M)
                __stcg(args.side + ((long long)m + args.side_qstride * q) * args.ld_side + c,
                       y * cscale);
              acc[j * 32 * kEpiWarps] = fma(y, hc, acc[j * 32 * kEpiWarps]);
            }
          }
          ew_final += prof_clock() - e2;
        }
        if (cval) {
          double* out = args.out + (args.S > 1 ? (long long)U.s * args.part_stride : 0LL);
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int m = mb + j;
            if (m < args.M) out[(long long)m * args.ldo + c] = acc[j * 32 * kEpiWarps];
          }
        }
      } else {
        // packed remainder tile: column n = half*32 + j holds slab qb + n / r,
        // row M - r + n % r.  Each column's Hi-weighted product is parked in
        // shared memory, then the half-0 warp of the quadrant sums the slabs
        // of every row in ascending order (deterministic, shape-only order).
        drain_pass(tfull, tempty, slab, trow, lane, P, ew_wait, ew_load);
        ++slab;
        const int r = args.rem_rows, nq = U.qe - U.qb;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int n = half * 32 + j, ql = n / r, m = U.m0 + n % r;
          double t = 0.0;
          if (ql < nq) {
            const int q = U.qb + ql;
            const int ex = __ldg(args.rex + (long long)q * args.M + m);
            const double y = exp_add(P[j], ex);
            if (kSide && cval)
              __stcg(args.side + ((long long)m + args.side_qstride * q) * args.ld_side + c,
                     side_fast ? exp_add(P[j], ex + kside) : y * cscale);
            if (cval) t = y * (__ldg(args.hi + (long long)q * args.ldh + c) * cscale);
          }
          acc[j * 32 * kEpiWarps] = t;
        }
        asm volatile("bar.sync %0, 64;" ::"r"(1 + quad) : "memory");
        if (half == 0 && cval) {
          double* out = args.out + (args.S > 1 ? (long long)U.s * args.part_stride : 0LL);
          for (int ml = 0; ml < r; ++ml) {
            double sum = 0.0;
            for (int ql = 0; ql < nq; ++ql) {
              const int n = ql * r + ml;
              sum += n < 32 ? acc[n * 32 * kEpiWarps] : acc[(n - 32) * 32 * kEpiWarps + 128];
            }
            out[(long long)(U.m0 + ml) * args.ldo + c] = sum;
          }
        }
        asm volatile("bar.sync %0, 64;" ::"r"(1 + quad) : "memory");
      }
    }
    if (kProfile && lane == 0 && (warp == 2 || warp == 5)) {
      // epilogue timing (warp 2: SMSP 2; warp 5: shares SMSP 1 with the MMA warp)
      unsigned long long* p = args.prof + 148 * 4 + (blockIdx.x * 2 + (warp == 5)) * 4;
      p[0] = prof_clock() - e_start;
      p[1] = ew_wait;
      p[2] = ew_load;
      p[3] = ew_final;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(kTmemCols));
  }
}

}  // namespace oz
}  // namespace cals
