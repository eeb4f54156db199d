// Accuracy of daba::log1p_pos (device_math.cuh) against the library log1p over q in [0, 1e300]: relative and ulp
// error on 2^24 log-uniform samples per decade band plus the special points.  Build and run on the B200:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I include -o tools/log1p_check tools/log1p_check.cu
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2305_07026_b200/csrc/device_math.cuh"

__global__ void k_check(double lo_exp, double hi_exp, int64_t n, unsigned long long* max_ulp, double* max_rel,
                        double* worst_q) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  // log-uniform q in [10^lo, 10^hi] (a counter-based hash for the fraction)
  uint64_t h = (uint64_t)i * 0x9E3779B97F4A7C15ull;
  h ^= h >> 31;
  h *= 0xBF58476D1CE4E5B9ull;
  h ^= h >> 29;
  const double t = (double)(h >> 11) * (1.0 / 9007199254740992.0);
  const double q = pow(10.0, lo_exp + (hi_exp - lo_exp) * t);
  const double a = daba::log1p_pos(q), b = log1p(q);
  const long long ua = __double_as_longlong(a), ub = __double_as_longlong(b);
  const unsigned long long d = (unsigned long long)(ua > ub ? ua - ub : ub - ua);
  const unsigned long long prev = atomicMax(max_ulp, d);
  if (d > prev) *worst_q = q;
  const double rel = b != 0.0 ? fabs(a - b) / fabs(b) : fabs(a);
  // (relative error as ordered bits of a non-negative double)
  atomicMax(reinterpret_cast<unsigned long long*>(max_rel), (unsigned long long)__double_as_longlong(rel));
}

int main() {
  unsigned long long* du;
  double *dr, *dq;
  cudaMalloc(&du, 8);
  cudaMalloc(&dr, 8);
  cudaMalloc(&dq, 8);
  const double bands[][2] = {{-300, -20}, {-20, -8}, {-8, -3}, {-3, -1}, {-1, -0.3827}, {-0.3827, -0.3828},
                             {-0.4, 0.0}, {0.0, 1.0}, {1.0, 3.0}, {3.0, 30.0}, {30.0, 300.0}};
  unsigned long long worst_all = 0;
  for (auto& b : bands) {
    cudaMemset(du, 0, 8);
    cudaMemset(dr, 0, 8);
    cudaMemset(dq, 0, 8);
    const int64_t n = 1 << 24;
    k_check<<<(unsigned)((n + 255) / 256), 256>>>(b[0], b[1], n, du, dr, dq);
    unsigned long long u;
    double r, q;
    cudaMemcpy(&u, du, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&r, dr, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&q, dq, 8, cudaMemcpyDeviceToHost);
    printf("q in [1e%g, 1e%g]: max %llu ulp, max rel %.3e (worst q %.17g)\n", b[0], b[1], u, r, q);
    if (u > worst_all) worst_all = u;
  }
  printf("max ulp over all bands: %llu (%s)\n", worst_all, cudaGetErrorString(cudaGetLastError()));
  return worst_all <= 4 ? 0 : 1;
}
