// Day-0 microbenchmarks for the DABA hot path on B200 (sm_100a):
//  1. FP64 FMA throughput (independent chains, full chip)
//  2. fp64 RED (atomicAdd without return) throughput to scattered addresses
//  3. 32-byte random gather bandwidth from a 143 MB buffer (point-state gather)
//  4. streaming copy bandwidth
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__global__ void fma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void red_kernel(double* acc, const int* idx, int64_t n, int per) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = t; i < n; i += stride) {
    int j = idx[i];
    for (int k = 0; k < per; ++k) atomicAdd(&acc[(int64_t)j * per + k], 1.0);
  }
}
__global__ void gather_kernel(const double4* pts, const int* idx, int64_t n, double* out) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  double s = 0;
  for (int64_t i = t; i < n; i += stride) { const double4 p = pts[idx[i]]; s += p.x + p.y + p.z; }
  if (s == 12345.0) out[0] = s;
}
__global__ void copy_kernel(const double2* a, double2* b, int64_t n) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = t; i < n; i += stride) b[i] = a[i];
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int l2; cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d  L2 %d B  clockRate %d kHz\n", sms, l2, clk);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  double* out; CK(cudaMalloc(&out, 1 << 24));
  // 1. FP64 FMA
  for (int rep = 0; rep < 3; ++rep) {
    int blocks = sms * 8, threads = 256, iters = 4000;
    cudaEventRecord(e0); fma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double fmas = (double)blocks * threads * iters * 64;
    printf("fp64 FMA: %.3f ms  %.2f TFMA/s = %.2f TFLOP/s  (%.1f FMA/clk/SM at %d MHz)\n", ms, fmas / ms / 1e9, 2 * fmas / ms / 1e9,
           fmas / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  }
  // 2. RED f64 scattered
  int64_t N = 4456117, n = 28987644;
  int* idx; CK(cudaMalloc(&idx, n * 4)); double* acc; CK(cudaMalloc(&acc, N * 8 * 8));
  int* h = (int*)malloc(n * 4); uint64_t s = 88172645463325252ull;
  for (int64_t i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = (int)(s % N); }
  CK(cudaMemcpy(idx, h, n * 4, cudaMemcpyHostToDevice));
  for (int per : {1, 4, 8}) for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); red_kernel<<<sms * 16, 256>>>(acc, idx, n, per); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("RED.f64 random pts, %d per obs: %.3f ms  %.1f G atom/s\n", per, ms, n * per / ms / 1e6);
  }
  // sorted indices (locality)
  for (int64_t i = 0; i < n; ++i) h[i] = (int)(i * N / n);
  CK(cudaMemcpy(idx, h, n * 4, cudaMemcpyHostToDevice));
  for (int per : {1, 8}) {
    cudaEventRecord(e0); red_kernel<<<sms * 16, 256>>>(acc, idx, n, per); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("RED.f64 sorted pts, %d per obs: %.3f ms  %.1f G atom/s\n", per, ms, n * per / ms / 1e6);
  }
  // 3. gather
  double4* pts; CK(cudaMalloc(&pts, N * 32)); cudaMemset(pts, 0, N * 32);
  s = 88172645463325252ull;
  for (int64_t i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = (int)(s % N); }
  CK(cudaMemcpy(idx, h, n * 4, cudaMemcpyHostToDevice));
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0); gather_kernel<<<sms * 16, 256>>>(pts, idx, n, out); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("gather 32B random of 143MB: %.3f ms  %.1f G/s  %.0f GB/s(32B sectors+idx)\n", ms, n / ms / 1e6, n * 36.0 / ms / 1e6);
  }
  // 4. copy
  int64_t cn = (int64_t)1 << 27; double2 *a, *b; CK(cudaMalloc(&a, cn * 16)); CK(cudaMalloc(&b, cn * 16));
  cudaMemset(a, 0, cn * 16);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0); copy_kernel<<<sms * 16, 256>>>(a, b, cn); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("copy 2 GiB: %.3f ms  %.0f GB/s\n", ms, 2.0 * cn * 16 / ms / 1e6);
  }
  return 0;
}
