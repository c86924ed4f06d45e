// tcgen05 kind::i8 probe for B200 (sm_100a): correctness of the hand-built
// shared-memory / instruction descriptors (SWIZZLE_32B and SWIZZLE_NONE K-major)
// against a CPU integer GEMM, MMA throughput for the shapes the Ozaki-sliced
// MTTKRP would use (M=128, N=16..128, SS and A-in-TMEM), and TMEM load throughput.
// Standalone: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_probe tc_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile("{\n.reg .pred P1;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra WAIT_%=;\n}\n"
               ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
               ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_i8_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n"
               ::"r"(d), "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

// smem matrix descriptor (sm100): start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46),
// version 1 [46,48), layout [61,64): 0 none, 6 swizzle-32B
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(layout & 7) << 61;
  return d;
}
// instruction descriptor kind::i8: c_format S32 (2) [4,6), a_format [7,10), b_format [10,13)
// (1 signed, 0 unsigned), K-major A/B, N>>3 [17,23), M>>4 [24,29)
__host__ __device__ constexpr uint32_t make_idesc(int M, int N, int a_signed, int b_signed) {
  return (2u << 4) | ((uint32_t)a_signed << 7) | ((uint32_t)b_signed << 10) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int NCOLS>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)), "n"(NCOLS));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
template <int NCOLS>
__device__ __forceinline__ void tmem_free(uint32_t addr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(addr), "n"(NCOLS));
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// byte offset of (row r, k byte) in a K-major tile of one 32-byte K step
__host__ __device__ inline uint32_t off_sw32(int r, int k) {
  uint32_t a = r * 32 + k;
  return a ^ (((a >> 7) & 1) << 4);
}
__host__ __device__ inline uint32_t off_none(int r, int k) {
  // core matrices 8 rows x 16 B; [rowgroup][kchunk(2)][8][16] -> LBO 128, SBO 256
  return (r >> 3) * 256 + (k >> 4) * 128 + (r & 7) * 16 + (k & 15);
}

// ---------------------------------------------------------------- correctness
// D[128][N] = A[128][K] * B[N][K]^T, K = 32*KS, int8 (a signed, b signed/unsigned)
template <int N>
__global__ void mma_check(const int8_t* A, const int8_t* B, int KS, int layout, int b_signed, int* D) {
  __shared__ __align__(1024) uint8_t sa[4][128 * 32];
  __shared__ __align__(1024) uint8_t sb[4][N * 32];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  for (int ks = 0; ks < KS; ++ks) {
    for (int i = tid; i < 128 * 32; i += blockDim.x) {
      int r = i / 32, k = i % 32;
      uint32_t o = layout == 6 ? off_sw32(r, k) : off_none(r, k);
      sa[ks][o] = (uint8_t)A[r * 32 * KS + ks * 32 + k];
    }
    for (int i = tid; i < N * 32; i += blockDim.x) {
      int r = i / 32, k = i % 32;
      uint32_t o = layout == 6 ? off_sw32(r, k) : off_none(r, k);
      sb[ks][o] = (uint8_t)B[r * 32 * KS + ks * 32 + k];
    }
  }
  if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  if (tid < 32) tmem_alloc<128>(&tbase);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t d = tbase;
  if (tid == 0) {
    const uint32_t lbo = layout == 6 ? 16 : 128, sbo = 256;
    for (int ks = 0; ks < KS; ++ks)
      mma_i8(d, make_desc(smem_u32(sa[ks]), lbo, sbo, layout), make_desc(smem_u32(sb[ks]), lbo, sbo, layout),
             make_idesc(128, N, 1, b_signed), ks > 0);
    tc_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const int warp = tid / 32;
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t r[16];
    tmem_ld16(d + ((uint32_t)(warp * 32) << 16) + c0, r);
    tmem_wait_ld();
    for (int j = 0; j < 16; ++j) D[tid * N + c0 + j] = (int)r[j];
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) tmem_free<128>(tbase);
}

// ---------------------------------------------------------------- throughput
// Each CTA issues iters x G x KS MMAs (M=128, N) into G accumulators; SS or TS.
template <int N, int G, bool TS>
__global__ void mma_rate(int iters, int* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sa = smem;                 // 8 K-steps of A: 8 x 4 KB
  uint8_t* sb = smem + 8 * 4096;      // 8 K-steps of B: 8 x N*32
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  for (int i = tid; i < 8 * 4096 + 8 * N * 32; i += blockDim.x) smem[i] = (uint8_t)(i * 7);
  if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  if (tid < 32) tmem_alloc<512>(&tbase);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t d = tbase;
  if (tid == 0) {
    const uint32_t idesc = make_idesc(128, N, 1, 0);
    const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
#pragma unroll
        for (int g = 0; g < G; ++g) {
          uint64_t bd = make_desc(b0 + ks * N * 32, 16, 256, 6);
          if (TS) {
            // A from TMEM: columns after the accumulators, 8 columns per 32-byte K step
            mma_i8_ts(d + g * N, d + G * N + ks * 8, bd, idesc, 1);
          } else {
            uint64_t ad = make_desc(a0 + ks * 4096, 16, 256, 6);
            mma_i8(d + g * N, ad, bd, idesc, 1);
          }
        }
      }
    }
    tc_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t r[16];
  tmem_ld16(d + ((uint32_t)((tid / 32) * 32) << 16), r);
  tmem_wait_ld();
  if (r[0] == 0x12345 && r[1] == 7) sink[0] = r[2];
  tc_fence_before();
  __syncthreads();
  if (tid < 32) tmem_free<512>(tbase);
}

// TMEM -> register load throughput: 4 warps (128 threads) read x16 chunks
__global__ void tmem_rate(int iters, int* sink) {
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  if (tid < 32) tmem_alloc<512>(&tbase);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t d = tbase + ((uint32_t)((tid / 32) * 32) << 16);
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 512; c += 64) {
      uint32_t r0[16], r1[16], r2[16], r3[16];
      tmem_ld16(d + c, r0);
      tmem_ld16(d + c + 16, r1);
      tmem_ld16(d + c + 32, r2);
      tmem_ld16(d + c + 48, r3);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 16; ++j) acc += r0[j] ^ r1[j] ^ r2[j] ^ r3[j];
    }
  }
  if (acc == 0x12345) sink[0] = acc;
  tc_fence_before();
  __syncthreads();
  if (tid < 32) tmem_free<512>(tbase);
}


template <int COL>
__device__ __forceinline__ void mma_i8_col(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if (COL == 0)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                 ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
  else if (COL == 1)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8.collector::a::fill [%0], %1, %2, %3, p;\n}\n"
                 ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
  else if (COL == 2)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8.collector::a::use [%0], %1, %2, %3, p;\n}\n"
                 ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
  else
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8.collector::a::lastuse [%0], %1, %2, %3, p;\n}\n"
                 ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

// the Ozaki pattern: 7 A slices x 7 B slices, products i+j<=6 (0-based), acc g=i+j
// USE_COL: A-slice-major order with collector fill/use/lastuse
template <int N, bool USE_COL>
__global__ void oz_pattern(int iters, int* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sa = smem;               // 7 x 4 KB
  uint8_t* sb = smem + 7 * 4096;    // 7 x N*32
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  for (int i = tid; i < 7 * 4096 + 7 * N * 32; i += blockDim.x) smem[i] = (uint8_t)(i * 7);
  if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  if (tid < 32) tmem_alloc<512>(&tbase);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t d = tbase;
  if (tid == 0) {
    const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 7; ++i) {
#pragma unroll
        for (int j = 0; j < 7 - i; ++j) {
          uint64_t ad = make_desc(a0 + i * 4096, 16, 256, 6);
          uint64_t bd = make_desc(b0 + j * N * 32, 16, 256, 6);
          uint32_t idesc = make_idesc(128, N, i == 0, j == 0);
          const int last = 6 - i;
          if (!USE_COL || last == 0) mma_i8_col<0>(d + (i + j) * N, ad, bd, idesc, 1);
          else if (j == 0) mma_i8_col<1>(d + (i + j) * N, ad, bd, idesc, 1);
          else if (j == last) mma_i8_col<3>(d + (i + j) * N, ad, bd, idesc, 1);
          else mma_i8_col<2>(d + (i + j) * N, ad, bd, idesc, 1);
        }
      }
    }
    tc_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t r[16];
  tmem_ld16(d + ((uint32_t)((tid / 32) * 32) << 16), r);
  tmem_wait_ld();
  if (r[0] == 0x12345 && r[1] == 7) sink[0] = r[2];
  tc_fence_before();
  __syncthreads();
  if (tid < 32) tmem_free<512>(tbase);
}

// correctness of the collector path: D_g = sum_{i+j=g} A_i B_j^T (one K step)
__global__ void oz_col_check(const int8_t* A, const int8_t* B, int* D) {
  __shared__ __align__(1024) uint8_t sa[7][128 * 32];
  __shared__ __align__(1024) uint8_t sb[7][64 * 32];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  for (int s = 0; s < 7; ++s) {
    for (int i = tid; i < 128 * 32; i += blockDim.x) sa[s][off_sw32(i / 32, i % 32)] = (uint8_t)A[s * 4096 + i];
    for (int i = tid; i < 64 * 32; i += blockDim.x) sb[s][off_sw32(i / 32, i % 32)] = (uint8_t)B[s * 2048 + i];
  }
  if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  if (tid < 32) tmem_alloc<512>(&tbase);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t d = tbase;
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < 7; ++i) {
#pragma unroll
      for (int j = 0; j < 7 - i; ++j) {
        uint64_t ad = make_desc(smem_u32(sa[i]), 16, 256, 6);
        uint64_t bd = make_desc(smem_u32(sb[j]), 16, 256, 6);
        uint32_t idesc = make_idesc(128, 64, i == 0, j == 0);
        const int last = 6 - i;
        const uint32_t acc = i > 0;
        if (last == 0) mma_i8_col<0>(d + (i + j) * 64, ad, bd, idesc, acc);
        else if (j == 0) mma_i8_col<1>(d + (i + j) * 64, ad, bd, idesc, acc);
        else if (j == last) mma_i8_col<3>(d + (i + j) * 64, ad, bd, idesc, acc);
        else mma_i8_col<2>(d + (i + j) * 64, ad, bd, idesc, acc);
      }
    }
    tc_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const int warp = tid / 32;
  for (int c0 = 0; c0 < 7 * 64; c0 += 16) {
    uint32_t r[16];
    tmem_ld16(d + ((uint32_t)(warp * 32) << 16) + c0, r);
    tmem_wait_ld();
    for (int j = 0; j < 16; ++j) D[tid * 448 + c0 + j] = (int)r[j];
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) tmem_free<512>(tbase);
}

static void col_check() {
  std::vector<int8_t> A(7 * 4096), B(7 * 2048);
  for (auto& v : A) v = (int8_t)(rand() % 256 - 128);
  for (auto& v : B) v = (int8_t)(rand() % 256 - 128);
  int8_t *dA, *dB; int* dD;
  CK(cudaMalloc(&dA, A.size())); CK(cudaMalloc(&dB, B.size())); CK(cudaMalloc(&dD, 128 * 448 * 4));
  CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
  oz_col_check<<<1, 128>>>(dA, dB, dD);
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  std::vector<int> D(128 * 448);
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int g = 0; g < 7; ++g)
    for (int r = 0; r < 128; ++r)
      for (int c = 0; c < 64; ++c) {
        long long s = 0;
        for (int i = 0; i <= g; ++i) {
          int j = g - i;
          for (int k = 0; k < 32; ++k) {
            int a = i == 0 ? (int)A[i * 4096 + r * 32 + k] : (int)(uint8_t)A[i * 4096 + r * 32 + k];
            int b = j == 0 ? (int)B[j * 2048 + c * 32 + k] : (int)(uint8_t)B[j * 2048 + c * 32 + k];
            s += a * b;
          }
        }
        if (s != D[r * 448 + g * 64 + c]) { if (bad < 4) printf("  col mismatch g%d (%d,%d) %d vs %lld\n", g, r, c, D[r * 448 + g * 64 + c], s); ++bad; }
      }
  printf("collector check: %s (%d bad)\n", bad ? "FAIL" : "ok", bad);
}

template <int N, bool COL>
static void pattern_rate(int sms) {
  int* sink; CK(cudaMalloc(&sink, 4));
  const int smem = 7 * 4096 + 7 * N * 32;
  CK(cudaFuncSetAttribute(oz_pattern<N, COL>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  oz_pattern<N, COL><<<sms, 128, smem>>>(10, sink);
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  const int iters = 400;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  oz_pattern<N, COL><<<sms, 128, smem>>>(iters, sink);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double cyc = ms * 1e-3 * clk * 1e3;
  printf("oz_pattern N=%d collector=%d: %.1f clk per MMA\n", N, (int)COL, cyc / (iters * 28.0));
  cudaFree(sink);
}


// issue-rate experiment: NW warps each issue a share of the 28 products
// (warp w takes products p with p % NW == w); warp-uniform loop + elect.sync
template <int N, int NW>
__global__ void oz_multi(int iters, int* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sa = smem;
  uint8_t* sb = smem + 7 * 4096;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < 7 * 4096 + 7 * N * 32; i += blockDim.x) smem[i] = (uint8_t)(i * 7);
  if (tid == 0) { mbar_init(&bar, NW); asm volatile("fence.mbarrier_init.release.cluster;"); }
  if (warp == 0) tmem_alloc<512>(&tbase);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t d = tbase;
  if (warp < NW) {
    const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb);
    const uint64_t da = make_desc(a0, 16, 256, 6), db = make_desc(b0, 16, 256, 6);
    for (int it = 0; it < iters; ++it) {
      int p = 0;
#pragma unroll
      for (int i = 0; i < 7; ++i) {
#pragma unroll
        for (int j = 0; j < 7 - i; ++j, ++p) {
          if (p % NW != warp) continue;
          uint32_t idesc = make_idesc(128, N, i == 0, j == 0);
          asm volatile("{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
                       "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(d + (i + j) * N), "l"(da + (uint64_t)(i * 256)), "l"(db + (uint64_t)(j * N * 2)), "r"(idesc), "r"(1) : "memory");
        }
      }
    }
    asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(&bar)) : "memory");
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t r[16];
  if (warp < 4) {
    tmem_ld16(d + ((uint32_t)((warp) * 32) << 16), r);
    tmem_wait_ld();
    if (r[0] == 0x12345 && r[1] == 7) sink[0] = r[2];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_free<512>(tbase);
}

template <int N, int NW>
static void multi_rate(int sms) {
  int* sink; CK(cudaMalloc(&sink, 4));
  const int smem = 7 * 4096 + 7 * N * 32;
  CK(cudaFuncSetAttribute(oz_multi<N, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  oz_multi<N, NW><<<sms, 128, smem>>>(10, sink);
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  const int iters = 400;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  oz_multi<N, NW><<<sms, 128, smem>>>(iters, sink);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double cyc = ms * 1e-3 * clk * 1e3;
  printf("oz_multi N=%d issuing warps=%d: %.1f clk per MMA\n", N, NW, cyc / (iters * 28.0));
  cudaFree(sink);
}


// pipeline ping-pong: producer warp <-> MMA warp over NST stages (no TMA),
// 28 MMAs per stage into 7 accumulators, commit per stage
template <int N, int NST>
__global__ void oz_pipe(int iters, int* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[8], empty[8], done;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32;
  const int stage_bytes = 7 * 4096 + 7 * N * 32;
  for (int i = tid; i < NST * stage_bytes; i += blockDim.x) smem[i] = (uint8_t)(i * 7);
  if (tid == 0) {
    for (int i = 0; i < NST; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    mbar_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) tmem_alloc<512>(&tbase);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t d = tbase;
  const int total = iters;
  if (warp == 1) {  // producer
    if ((tid & 31) == 0) {
      int st = 0; uint32_t ph = 0;
      for (int k = 0; k < total; ++k) {
        mbar_wait(&empty[st], ph ^ 1);
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[st])) : "memory");
        if (++st == NST) { st = 0; ph ^= 1; }
      }
    }
  } else if (warp == 0) {  // MMA
    int st = 0; uint32_t ph = 0;
    const uint64_t sd = make_desc(smem_u32(smem), 16, 256, 6);
    for (int k = 0; k < total; ++k) {
      mbar_wait(&full[st], ph);
      tc_fence_after();
      const uint64_t a0 = sd + (uint64_t)((st * stage_bytes) >> 4);
      const uint64_t b0 = a0 + (uint64_t)((7 * 4096) >> 4);
#pragma unroll
      for (int i = 0; i < 7; ++i)
#pragma unroll
        for (int j = 0; j < 7 - i; ++j) {
          uint32_t idesc = make_idesc(128, N, i == 0, j == 0);
          asm volatile("{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
                       "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(d + (i + j) * N), "l"(a0 + (uint64_t)(i * 256)), "l"(b0 + (uint64_t)(j * N * 2)), "r"(idesc), "r"(1) : "memory");
        }
      asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(&empty[st])) : "memory");
      if (++st == NST) { st = 0; ph ^= 1; }
    }
    asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(&done)) : "memory");
  }
  mbar_wait(&done, 0);
  tc_fence_after();
  uint32_t r[16];
  if (warp < 4) {
    tmem_ld16(d + ((uint32_t)(warp * 32) << 16), r);
    tmem_wait_ld();
    if (r[0] == 0x12345 && r[1] == 7) sink[0] = r[2];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_free<512>(tbase);
}

template <int N, int NST>
static void pipe_rate(int sms) {
  int* sink; CK(cudaMalloc(&sink, 4));
  const int smem = NST * (7 * 4096 + 7 * N * 32);
  CK(cudaFuncSetAttribute(oz_pipe<N, NST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  oz_pipe<N, NST><<<sms, 128, smem>>>(10, sink);
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  const int iters = 400;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  oz_pipe<N, NST><<<sms, 128, smem>>>(iters, sink);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double cyc = ms * 1e-3 * clk * 1e3;
  printf("oz_pipe N=%d stages=%d: %.1f clk per MMA\n", N, NST, cyc / (iters * 28.0));
  cudaFree(sink);
}


// FP64 throughput of DFMA warps while one warp streams INT8 MMAs (MMA=1) or not
template <bool MMA, int OP>
__global__ void dfma_vs_mma(int iters, int dfma_iters, int* sink, double* dsink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < 7 * 4096 + 7 * 64 * 32; i += blockDim.x) smem[i] = (uint8_t)(i * 7);
  if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  if (warp == 0) tmem_alloc<512>(&tbase);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t d = tbase;
  if (warp == 0) {
    if (MMA) {
      const uint64_t da = make_desc(smem_u32(smem), 16, 256, 6), db = make_desc(smem_u32(smem) + 7 * 4096, 16, 256, 6);
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 7; ++i)
#pragma unroll
          for (int j = 0; j < 7 - i; ++j) {
            uint32_t idesc = make_idesc(128, 64, i == 0, j == 0);
            asm volatile("{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
                         "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                         ::"r"(d + (i + j) * 64), "l"(da + (uint64_t)(i * 256)), "l"(db + (uint64_t)(j * 128)), "r"(idesc), "r"(1) : "memory");
          }
      }
    }
    asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(&bar)) : "memory");
  } else if (warp >= 2) {
    if (OP == 0) {
      double a[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = tid * 1e-3 + k;
      const double b = 1.0000001, c = 1e-9;
      for (int it = 0; it < dfma_iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
      }
      double s = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) s += a[k];
      if (s == 12345.0) dsink[0] = s;
    } else if (OP == 1) {
      float a[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = tid * 1e-3f + k;
      for (int it = 0; it < dfma_iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fmaf(a[k], 1.0000001f, 1e-9f);
      }
      float s = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) s += a[k];
      if (s == 12345.0f) dsink[0] = s;
    } else if (OP == 2) {
      unsigned a[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = tid + k;
      for (int it = 0; it < dfma_iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = a[k] * 747796405u + 2891336453u;
      }
      unsigned s = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) s += a[k];
      if (s == 12345u) dsink[0] = s;
    } else {
      double a[8];
      int v = tid;
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = 0;
      for (int it = 0; it < dfma_iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) { a[k] += (double)(v + k * it); }
      }
      double s = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) s += a[k];
      if (s == 12345.0) dsink[0] = s;
    }
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_free<512>(tbase);
}

template <int OP>
static void dfma_mma_test(int sms) {
  int* sink; double* dsink; CK(cudaMalloc(&sink, 4)); CK(cudaMalloc(&dsink, 8));
  const int smem = 7 * 4096 + 7 * 64 * 32;
  CK(cudaFuncSetAttribute(dfma_vs_mma<true, OP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(dfma_vs_mma<false, OP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float t[3];
  for (int mode = 0; mode < 3; ++mode) {
    const int iters = mode == 0 ? 0 : 400, di = mode == 1 ? 0 : (OP == 1 || OP == 2 ? 80000 : 20000);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) dfma_vs_mma<false, OP><<<sms, 320, smem>>>(iters, di, sink, dsink);
      else dfma_vs_mma<true, OP><<<sms, 320, smem>>>(iters, di, sink, dsink);
      cudaEventRecord(e1);
      CK(cudaDeviceSynchronize());
      cudaEventElapsedTime(&t[mode], e0, e1);
    }
  }
  printf("op %d (0 dfma,1 ffma,2 imad,3 i2f.f64): alone %.3f ms, mma alone %.3f ms, both %.3f ms\n", OP, t[0], t[1], t[2]);
}

template <int N>
static bool check(int KS, int layout, int b_signed) {
  std::vector<int8_t> A(128 * 32 * KS), B(N * 32 * KS);
  for (auto& v : A) v = (int8_t)(rand() % 256 - 128);
  for (auto& v : B) v = (int8_t)(rand() % 256 - 128);
  int8_t *dA, *dB; int* dD;
  CK(cudaMalloc(&dA, A.size())); CK(cudaMalloc(&dB, B.size())); CK(cudaMalloc(&dD, 128 * N * 4));
  CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
  CK(cudaMemset(dD, 0, 128 * N * 4));
  mma_check<N><<<1, 128>>>(dA, dB, KS, layout, b_signed, dD);
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  std::vector<int> D(128 * N);
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < N; ++j) {
      long long s = 0;
      for (int k = 0; k < 32 * KS; ++k) {
        int a = A[i * 32 * KS + k];
        int b = b_signed ? (int)B[j * 32 * KS + k] : (int)(uint8_t)B[j * 32 * KS + k];
        s += a * b;
      }
      if (s != D[i * N + j]) { if (bad < 4) printf("  mismatch (%d,%d) gpu %d cpu %lld\n", i, j, D[i * N + j], s); ++bad; }
    }
  printf("check N=%d KS=%d layout=%s b_%s: %s (%d bad)\n", N, KS, layout == 6 ? "sw32" : "none",
         b_signed ? "s8" : "u8", bad ? "FAIL" : "ok", bad);
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
  return bad == 0;
}

template <int N, int G, bool TS>
static void rate(int sms) {
  int* sink; CK(cudaMalloc(&sink, 4));
  const int smem = 8 * 4096 + 8 * N * 32;
  CK(cudaFuncSetAttribute(mma_rate<N, G, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int iters = 400;
  mma_rate<N, G, TS><<<sms, 128, smem>>>(10, sink);
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mma_rate<N, G, TS><<<sms, 128, smem>>>(iters, sink);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double macs = (double)sms * iters * 8 * G * 128.0 * N * 32;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double cyc = ms * 1e-3 * clk * 1e3;
  printf("mma_rate N=%3d G=%d %s: %.3f ms  %.0f TOPS  %.0f MAC/clk/SM (at %d MHz)\n", N, G, TS ? "TS" : "SS",
         ms, 2 * macs / (ms * 1e-3) / 1e12, macs / sms / cyc, clk / 1000);
  cudaFree(sink);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  bool ok = true;
  printf("== descriptor / layout checks vs CPU integer GEMM\n");
  ok &= check<32>(1, 6, 1);
  ok &= check<32>(1, 0, 1);
  ok &= check<32>(4, 6, 0);
  ok &= check<64>(3, 6, 1);
  ok &= check<128>(2, 6, 0);
  ok &= check<16>(2, 6, 1);
  if (!ok) printf("DESCRIPTOR CHECK FAILED\n");
  printf("== MMA instruction rate (M=128, K=32, G accumulators, all SMs)\n");
  rate<16, 7, false>(sms);
  rate<32, 7, false>(sms);
  rate<48, 7, false>(sms);
  rate<64, 7, false>(sms);
  rate<128, 3, false>(sms);
  rate<256, 1, false>(sms);
  rate<16, 7, true>(sms);
  rate<32, 7, true>(sms);
  rate<64, 4, true>(sms);
  printf("== Ozaki pattern (28 products, 7 accumulators), issue warps, pipeline ping-pong\n");
  pattern_rate<64, false>(sms);
  multi_rate<64, 1>(sms);
  multi_rate<64, 2>(sms);
  pipe_rate<64, 2>(sms);
  pipe_rate<64, 3>(sms);
  printf("== other pipes concurrent with the INT8 MMA stream (time alone / MMA alone / both)\n");
  dfma_mma_test<0>(sms);
  dfma_mma_test<1>(sms);
  dfma_mma_test<2>(sms);
  dfma_mma_test<3>(sms);
  return 0;
}
