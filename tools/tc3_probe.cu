// A-operand-in-TMEM ("TS") INT8 MMA probe (B200, sm_100a).
// 1) correctness: tcgen05.cp (128x256b, SW32 K-major descriptor) of an smem
//    A tile into TMEM + TS MMA gives the same accumulators as the SS MMA, with
//    a single A buffer overwritten every K step (mma -> cp ordering).
// 2) rate: 7 Ozaki groups (28 products per K step, i + j <= 8) of N columns;
//    A slices copied into TMEM once per K step (7 cp) vs read by every MMA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc3_probe tc3_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(256 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)6 << 61);
}
__host__ __device__ constexpr uint32_t idesc(int N, int as, int bs) {
  return (2u << 4) | ((uint32_t)as << 7) | ((uint32_t)bs << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d), "r"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void cp128(uint32_t t, uint64_t s) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(t), "l"(s) : "memory");
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t ph) {
  asm volatile("{\n.reg .pred P1;\nW: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}\n" ::"r"(smem_u32(bar)), "r"(ph) : "memory");
}
__device__ __forceinline__ void tld(uint32_t t, uint32_t (&v)[32]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                 "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                 "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                 "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
               : "r"(t));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// --- 1: correctness (one CTA, 128 threads) ----------------------------------
__global__ void check_ts(int* bad, int* sample) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sa = smem;              // 4 K steps x 4 KB
  uint8_t* sb = smem + 4 * 4096;   // 4 K steps x 64 rows x 32 B
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32;
  uint32_t x = 12345u + tid * 7919u;
  for (int i = tid; i < 4 * 4096 + 4 * 2048; i += 128) { x = x * 1664525u + 1013904223u; smem[i] = (uint8_t)(x >> 24); }
  if (tid == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t t = tbase;
  if (warp == 0 && tid == 0) {
    const uint32_t id = idesc(64, 1, 0);
    for (int ks = 0; ks < 4; ++ks) {
      const uint64_t da = make_desc(smem_u32(sa + ks * 4096)), db = make_desc(smem_u32(sb + ks * 2048));
      mma_ss(t + 0, da, db, id, ks > 0);
      cp128(t + 256, da);                        // A -> TMEM cols 256..263 (one buffer)
      mma_ts(t + 64, t + 256, db, id, ks > 0);
    }
    commit(&bar);
  }
  wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t v0[32], v1[32];
  int nb = 0;
  for (int h = 0; h < 2; ++h) {
    tld(t + ((uint32_t)(warp * 32) << 16) + h * 32, v0);
    tld(t + ((uint32_t)(warp * 32) << 16) + 64 + h * 32, v1);
    for (int j = 0; j < 32; ++j) nb += v0[j] != v1[j];
    if (tid == 5 && h == 0) for (int j = 0; j < 4; ++j) { sample[j] = v0[j]; sample[4 + j] = v1[j]; }
  }
  atomicAdd(bad, nb);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
}

// --- 2: rate ------------------------------------------------------------------
// MODE 0: SS (A read from smem by every MMA); 1: TS with 7 cp per K step into
// NB A buffers; 2: TS without cp (A static in TMEM)
template <int N, int MODE, int NB, int CM = 0, int RND = 0>
__global__ void rate(int iters, int* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sa = smem;                  // 7 slices x 4 KB (one K step)
  uint8_t* sb = smem + 7 * 4096;       // 7 slices x N rows x 32 B
  __shared__ uint64_t bar, cbar[8];
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32;
  {
    uint32_t x = 2654435761u * (tid + 1) + blockIdx.x;
    for (int i = tid; i < 7 * 4096 + 7 * N * 32; i += blockDim.x) {
      x = x * 1664525u + 1013904223u;
      smem[i] = RND ? (uint8_t)(x >> 24) : (uint8_t)(i * 13);
    }
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&cbar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t t = tbase;
  const uint32_t abase = t + 7 * N;  // A buffers after the 7 accumulators
  if (tid == 0) {
    const uint64_t da = make_desc(smem_u32(sa)), db = make_desc(smem_u32(sb));
    for (int it = 0; it < iters; ++it) {
      for (int ks = 0; ks < 8; ++ks) {
        const uint32_t ab = abase + (uint32_t)((ks % NB) * 56);
        if (MODE == 1)
#pragma unroll
          for (int i = 0; i < 7; ++i) cp128(ab + i * 8, da + (uint64_t)(i * 256));
#pragma unroll
        for (int o1 = 0; o1 < 7; ++o1)
#pragma unroll
          for (int o2 = 1; o2 <= 7; ++o2) {
            // MODE 3: i-major order (same A slice for consecutive products)
            const int g = MODE == 3 ? o1 + o2 - 1 : o1;
            const int i = MODE == 3 ? o1 + 1 : o2;
            const int j = g + 2 - i;
            if (MODE == 3 && g > 6) continue;
            if (j < 1 || j > 7) continue;
            const uint32_t id = idesc(N, i == 1, j == 1);
            if (MODE == 0 || MODE == 3) mma_ss(t + g * N, da + (uint64_t)((i - 1) * 256), db + (uint64_t)((j - 1) * N * 2), id, 1);
            else mma_ts(t + g * N, ab + (i - 1) * 8, db + (uint64_t)((j - 1) * N * 2), id, 1);
            if ((CM & 2) && ks == 7 && i == (g + 1 < 7 ? g + 1 : 7)) commit(&cbar[g]);
          }
        if (CM & 1) commit(&cbar[7]);
      }
    }
    commit(&bar);
  }
  wait(&bar, 0);
  if (tid == 0 && iters < 0) sink[0] = t;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
}

template <int N, int MODE, int NB, int CM = 0, int RND = 0>
int run(int sms, const char* name) {
  int* sink; CK(cudaMalloc(&sink, 4));
  const int smem = 7 * 4096 + 7 * N * 32;
  CK(cudaFuncSetAttribute(rate<N, MODE, NB, CM, RND>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  rate<N, MODE, NB, CM, RND><<<sms, 128, smem>>>(10, sink);
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 300;
  cudaEventRecord(e0);
  rate<N, MODE, NB, CM, RND><<<sms, 128, smem>>>(iters, sink);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double cyc = ms * 1e-3 * clk * 1e3, nmma = (double)iters * 8 * 28;
  printf("%-28s N=%3d: %.1f clk per MMA, %.0f MAC/clk/SM, 28-product K step %.0f clk\n", name, N, cyc / nmma,
         128.0 * N * 32 * nmma / cyc, cyc / (iters * 8.0));
  return 0;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int *bad, *sample; CK(cudaMalloc(&bad, 4)); CK(cudaMalloc(&sample, 32)); CK(cudaMemset(bad, 0, 4));
  CK(cudaFuncSetAttribute(check_ts, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 4096));
  check_ts<<<1, 128, 6 * 4096>>>(bad, sample);
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  int hb, hs[8]; cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost); cudaMemcpy(hs, sample, 32, cudaMemcpyDeviceToHost);
  printf("TS vs SS mismatches: %d of 8192  (sample ss %d %d %d %d  ts %d %d %d %d)\n", hb, hs[0], hs[1], hs[2], hs[3], hs[4], hs[5], hs[6], hs[7]);
  run<64, 0, 1>(sms, "SS");
  run<64, 3, 1>(sms, "SS i-major order");
  run<64, 0, 1, 0, 1>(sms, "SS random data");
  run<64, 0, 1, 1>(sms, "SS + commit per K step");
  run<64, 0, 1, 2>(sms, "SS + 7 group commits / 8 K");
  run<64, 0, 1, 3>(sms, "SS + both");
  run<64, 1, 1>(sms, "TS + 7 cp, 1 A buffer");
  run<64, 2, 1>(sms, "TS, no cp");
  run<48, 0, 1>(sms, "SS");
  run<48, 1, 2>(sms, "TS + 7 cp, 2 A buffers");
  run<48, 2, 1>(sms, "TS, no cp");
  run<32, 0, 1>(sms, "SS");
  run<32, 1, 2>(sms, "TS + 7 cp, 2 A buffers");
  run<32, 2, 1>(sms, "TS, no cp");
  return 0;
}
