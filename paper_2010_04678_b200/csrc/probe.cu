// Diagnostics: live FP64 tensor-core (DMMA.8x8x4) peak and INT8 tcgen05
// peak of this GPU, the roofline denominators of the two fused-MTTKRP
// kernels in bench.py (MEASURED_PEAKS.json carries neither figure).
#include "internal.h"
#include "tcgen05.cuh"

#include <mutex>

namespace cals {

__global__ void dmma_peak_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double acc[8][2];
#pragma unroll
  for (int c = 0; c < 8; ++c) acc[c][0] = acc[c][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) dmma_8x8x4(acc[c][0], acc[c][1], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.0) out[0] = s;
}

// INT8 tensor-core peak: one CTA per SM streams tcgen05.mma kind::i8
// (M = 128, N = 256, K = 32, A/B from shared memory) into one TMEM
// accumulator -- the largest single-CTA instruction shape.
__global__ void __launch_bounds__(128, 1) i8_peak_kernel(int iters, int* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];  // 8 K steps of A (4 KB) and B (8 KB)
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 8 * (4096 + 8192); i += blockDim.x) sm[i] = (unsigned char)(i * 7);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  oz::tc_fence_before();
  __syncthreads();
  oz::tc_fence_after();
  const uint32_t d = tbase;
  if (warp == 0) {
    const uint32_t idesc = (2u << 4) | (1u << 7) | (0u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
    const uint64_t a0 = oz::desc_sw32(smem_u32(sm)), b0 = oz::desc_sw32(smem_u32(sm) + 8 * 4096);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int ks = 0; ks < 8; ++ks)
        oz::mma_i8_elect(d, a0 + (uint64_t)(ks * 256), b0 + (uint64_t)(ks * 512), idesc, 1u);
    }
    oz::tc_commit_elect(&bar);
  }
  mbar_wait(&bar, 0);
  oz::tc_fence_after();
  if (warp == 0 && tid == 0 && iters < 0) sink[0] = (int)d;
  oz::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    oz::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(d));
  }
}

}  // namespace cals

extern "C" int cals_int8_peak_probe(void* stream, double* tops) {
  using namespace cals;
  CALS_CHECK(tops, kErrInvalid, "null argument");
  int dev = 0;
  CALS_CUDA_TRY(cudaGetDevice(&dev));
  const int sms = sm_count(dev);
  cudaStream_t s = (cudaStream_t)stream;
  const int smem = 8 * (4096 + 8192);
  static std::once_flag once;
  static cudaError_t attr = cudaSuccess;
  std::call_once(once, [&] {
    attr = cudaFuncSetAttribute(i8_peak_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  });
  CALS_CUDA_TRY(attr);
  int* d = nullptr;
  CALS_CUDA_TRY(cudaMallocAsync(&d, 4, s));
  cudaEvent_t e0, e1;
  CALS_CUDA_TRY(cudaEventCreate(&e0));
  CALS_CUDA_TRY(cudaEventCreate(&e1));
  const int iters = 2000;
  i8_peak_kernel<<<sms, 128, smem, s>>>(50, d);
  CALS_CUDA_TRY(cudaEventRecord(e0, s));
  i8_peak_kernel<<<sms, 128, smem, s>>>(iters, d);
  CALS_CUDA_TRY(cudaEventRecord(e1, s));
  CALS_CUDA_TRY(cudaEventSynchronize(e1));
  float ms = 0.f;
  CALS_CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  CALS_CUDA_TRY(cudaFreeAsync(d, s));
  // 2 ops per MAC; 128 x 256 x 32 MACs per instruction, 8 per iteration
  *tops = double(sms) * iters * 8 * 2.0 * 128 * 256 * 32 / (ms * 1e-3) / 1e12;
  return kOk;
}

extern "C" int cals_fp64_peak_probe(void* stream, double* tflops) {
  using namespace cals;
  CALS_CHECK(tflops, kErrInvalid, "null argument");
  int dev = 0;
  CALS_CUDA_TRY(cudaGetDevice(&dev));
  const int sms = sm_count(dev);
  cudaStream_t s = (cudaStream_t)stream;
  double* d = nullptr;
  CALS_CUDA_TRY(cudaMallocAsync(&d, 8, s));
  cudaEvent_t e0, e1;
  CALS_CUDA_TRY(cudaEventCreate(&e0));
  CALS_CUDA_TRY(cudaEventCreate(&e1));
  const int iters = 20000, warps = 8;
  dmma_peak_kernel<<<sms, 32 * warps, 0, s>>>(d, 200);
  CALS_CUDA_TRY(cudaEventRecord(e0, s));
  dmma_peak_kernel<<<sms, 32 * warps, 0, s>>>(d, iters);
  CALS_CUDA_TRY(cudaEventRecord(e1, s));
  CALS_CUDA_TRY(cudaEventSynchronize(e1));
  float ms = 0.f;
  CALS_CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  CALS_CUDA_TRY(cudaFreeAsync(d, s));
  *tflops = double(sms) * warps * iters * 8 * 512.0 / (ms * 1e-3) / 1e12;
  return kOk;
}
