// Microbenchmark: FP64 throughput of DFMA vs mma.sync m8n8k4 f64 (DMMA) on this GPU (independent chains).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters) {
  double a[8];
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
  const double x = 1.000001, y = 1e-9;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], x, y);
  double s = 0;
  for (int k = 0; k < 8; ++k) s += a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dmma(double* out, int iters) {
  double c[4][2];
  for (int k = 0; k < 4; ++k) c[k][0] = c[k][1] = threadIdx.x * 1e-3 + k;
  const double a = 1.000001 + threadIdx.x * 1e-9, b = 1e-9 * threadIdx.x;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  double s = 0;
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// Half the warps run the DFMA chains, half a quarter of the DMMA chains (alone, each half takes about the same
// time): if the two share one FP64 pipe the time is the sum of the halves, if they run on separate units the max.
__global__ void k_mixed(double* out, int iters) {
  double s = 0;
  if ((threadIdx.x >> 5) & 1) {
    double c[4][2];
    for (int k = 0; k < 4; ++k) c[k][0] = c[k][1] = threadIdx.x * 1e-3 + k;
    const double a = 1.000001 + threadIdx.x * 1e-9, b = 1e-9 * threadIdx.x;
    for (int i = 0; i < iters / 4; ++i)  // a quarter of the chain: alone each half takes about as long
#pragma unroll
      for (int k = 0; k < 4; ++k)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  } else {
    double a[8];
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
    const double x = 1.000001, y = 1e-9;
    for (int i = 0; i < iters; ++i)
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = fma(a[k], x, y);
    for (int k = 0; k < 8; ++k) s += a[k];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  double* d;
  cudaMalloc(&d, sizeof(double) * blocks * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fmas = (double)blocks * threads * iters * 8;
    printf("DFMA: %.3f ms, %.2f T FMA/s\n", ms, fmas / ms / 1e9);
    cudaEventRecord(e0);
    k_dmma<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double mfmas = (double)blocks * (threads / 32) * iters * 4 * 256;  // 8x8x4 = 256 FMA per warp-MMA
    printf("DMMA m8n8k4: %.3f ms, %.2f T FMA/s  (%s)\n", ms, mfmas / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
    cudaEventRecord(e0);
    k_mixed<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("mixed (half the warps each): %.3f ms, %.2f T FMA/s  (%s)\n", ms, (fmas + mfmas / 4) / 2 / ms / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
