// cta_group::2 INT8 MMA rate probe (B200, sm_100a): does a CTA pair issuing
// M=256 x N x K=32 (each SM its 128 rows) beat the ~56 clk per M=128 N=64
// single-CTA instruction?  G accumulators of N columns, 8 K steps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc2_probe tc2_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(256 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)6 << 61);
}
__host__ __device__ constexpr uint32_t idesc(int M, int N) {
  return (2u << 4) | (1u << 7) | (0u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int N, int G, int CG>
__global__ void __cluster_dims__(2, 1, 1) mma_rate2(int iters, int* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sa = smem;                        // 8 x 4 KB (128 rows)
  uint8_t* sb = smem + 8 * 4096;             // 8 x (N/CG rows x 32 B)
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < 8 * 4096 + 8 * (N / CG) * 32; i += blockDim.x) smem[i] = (uint8_t)(i * 7);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    if (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t d = tbase;
  const uint32_t rank = cta_rank();
  const bool issuer = (CG == 1) || rank == 0;
  if (warp == 0 && issuer) {
    const uint64_t da = make_desc(smem_u32(sa)), db = make_desc(smem_u32(sb));
    const uint32_t id = idesc(128 * CG, N);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int ks = 0; ks < 8; ++ks)
#pragma unroll
        for (int g = 0; g < G; ++g) {
          if (CG == 2)
            asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
                         "@e tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, 1;\n}\n"
                         ::"r"(d + g * N), "l"(da + (uint64_t)(ks * 256)), "l"(db + (uint64_t)(ks * (N / CG) * 2)), "r"(id) : "memory");
          else
            asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
                         "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 1;\n}\n"
                         ::"r"(d + g * N), "l"(da + (uint64_t)(ks * 256)), "l"(db + (uint64_t)(ks * N * 2)), "r"(id) : "memory");
        }
    }
    if (CG == 2)
      asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
                   "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}\n"
                   ::"r"(smem_u32(&bar)), "h"((uint16_t)3) : "memory");
    else
      asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
                   "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n"
                   ::"r"(smem_u32(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred P1;\nW: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(smem_u32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0 && iters < 0) sink[0] = d;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();
  if (warp == 0) {
    if (CG == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(d));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(d));
  }
}

template <int N, int G, int CG>
int run(int sms) {
  int* sink; CK(cudaMalloc(&sink, 4));
  const int smem = 8 * 4096 + 8 * (N / CG) * 32;
  CK(cudaFuncSetAttribute(mma_rate2<N, G, CG>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int grid = sms / 2 * 2;
  mma_rate2<N, G, CG><<<grid, 128, smem>>>(10, sink);
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 400;
  cudaEventRecord(e0);
  mma_rate2<N, G, CG><<<grid, 128, smem>>>(iters, sink);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double cyc = ms * 1e-3 * clk * 1e3;
  // per SM: each instruction does 128 x N x 32 MACs on this SM
  const double per_sm_instr = (double)iters * 8 * G * (CG == 2 ? 1.0 : 1.0);
  printf("cta_group::%d N=%3d G=%d: %.1f clk per instruction per SM  (%.0f MAC/clk/SM)\n", CG, N, G,
         cyc / per_sm_instr, 128.0 * N * 32 * per_sm_instr / cyc);
  return 0;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<64, 7, 1>(sms);
  run<64, 7, 2>(sms);
  run<128, 3, 2>(sms);
  run<32, 7, 2>(sms);
  // candidates for a wider Ozaki tile (groups split over passes)
  run<128, 4, 1>(sms);
  run<128, 4, 2>(sms);
  run<112, 4, 1>(sms);
  run<112, 4, 2>(sms);
  run<96, 5, 1>(sms);
  run<96, 5, 2>(sms);
  run<256, 2, 1>(sms);
  run<256, 2, 2>(sms);
  return 0;
}
