// Diagnostics: live FP64 tensor-core (DMMA.8x8x4) peak of this GPU, used as
// the roofline denominator of the fused MTTKRP in bench.py (MEASURED_PEAKS.json
// carries no FP64 figure).  Independent chains, 8 warps per SM.
#include "internal.h"

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

}  // namespace cals

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
