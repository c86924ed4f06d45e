// FP64 peak probe for B200 (sm_100a): DMMA (mma.sync f64) vs DFMA vs DMMA+DMUL mix.
// Standalone: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double acc[CHAINS][2];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) { acc[c][0] = 0; acc[c][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.0) out[0] = s;
}

template <int CHAINS>
__global__ void dmma_mul_loop(double* out, int iters, int nmul) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double acc[CHAINS][2];
  double m[4] = {a, b, a * b, a + b};
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) { acc[c][0] = 0; acc[c][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a), "d"(b));
    }
    // nmul DMULs per CHAINS DMMAs (runtime so the compiler cannot fold)
#pragma unroll 4
    for (int j = 0; j < nmul; ++j) {
      asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(m[j & 3]) : "d"(b));
    }
  }
  double s = m[0] + m[1] + m[2] + m[3];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.0) out[0] = s;
}

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters) {
  double acc[CHAINS];
  double a = 1.0 + threadIdx.x * 1e-12, b = 0.999999;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(acc[c]) : "d"(b), "d"(a));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.0) out[0] = s;
}

int main() {
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* d; CK(cudaMalloc(&d, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  printf("SMs %d\n", sms);
  const int iters = 20000;
  for (int warps : {1, 2, 4, 8, 16, 32}) {
    int threads = 32 * warps;
    dmma_loop<8><<<sms, threads>>>(d, 100);
    CK(cudaEventRecord(e0));
    dmma_loop<8><<<sms, threads>>>(d, iters);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = (double)sms * warps * iters * 8 * 512.0;
    printf("DMMA m8n8k4 warps/SM=%2d chains=8: %.2f TFLOP/s (%.3f ms)\n", warps, flops / ms / 1e9, ms);
  }
  for (int warps : {4, 8, 16}) {
    int threads = 32 * warps;
    dmma_loop<2><<<sms, threads>>>(d, 100);
    CK(cudaEventRecord(e0));
    dmma_loop<2><<<sms, threads>>>(d, iters * 4);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = (double)sms * warps * iters * 4 * 2 * 512.0;
    printf("DMMA m8n8k4 warps/SM=%2d chains=2: %.2f TFLOP/s\n", warps, flops / ms / 1e9);
  }
  for (int warps : {4, 8, 16, 32}) {
    int threads = 32 * warps;
    dfma_loop<8><<<sms, threads>>>(d, 100);
    CK(cudaEventRecord(e0));
    dfma_loop<8><<<sms, threads>>>(d, iters);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = (double)sms * threads * iters * 8 * 2.0;
    printf("DFMA warps/SM=%2d chains=8: %.2f TFLOP/s\n", warps, flops / ms / 1e9);
  }
  for (int nmul : {0, 1, 2, 4, 8, 16, 32}) {
    int warps = 8, threads = 256;
    dmma_mul_loop<8><<<sms, threads>>>(d, 100, nmul);
    CK(cudaEventRecord(e0));
    dmma_mul_loop<8><<<sms, threads>>>(d, iters, nmul);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = (double)sms * warps * iters * 8 * 512.0;
    printf("DMMA(8)+%2d DMUL per iter, 8 warps/SM: DMMA %.2f TFLOP/s\n", nmul, flops / ms / 1e9);
  }
  CK(cudaGetLastError());
  return 0;
}
