// MUFU.RSQ64H (rsqrt.approx.ftz.f64) accuracy and throughput on B200 (development aid).
// Prints max |e| with e = 1 - x*y^2 over 2^24 log-uniform x in [1e-6, 1e6], and the
// raw MUFU throughput per SM per clock.
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

__device__ __forceinline__ double rsq_seed(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

__global__ void acc_kernel(unsigned long long* maxbits, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double u = (i + 0.5) / n;
  double x = exp(log(1e-6) + u * (log(1e6) - log(1e-6)));
  double y = rsq_seed(x);
  double e = fabs(fma(-x, y * y, 1.0));
  atomicMax(maxbits, (unsigned long long)__double_as_longlong(e));
}

__global__ void thr_kernel(double* out, int iters) {
  double x[8], acc[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) { x[c] = 1.0 + threadIdx.x * 1e-3 + c; acc[c] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] = rsq_seed(acc[c] + x[c]);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

int main() {
  unsigned long long* mb;
  cudaMalloc(&mb, 8);
  cudaMemset(mb, 0, 8);
  int n = 1 << 24;
  acc_kernel<<<n / 256, 256>>>(mb, n);
  unsigned long long h;
  cudaMemcpy(&h, mb, 8, cudaMemcpyDeviceToHost);
  double emax;
  memcpy(&emax, &h, 8);
  cudaDeviceProp pr;
  cudaGetDeviceProperties(&pr, 0);
  double* out;
  cudaMalloc(&out, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int blocks = pr.multiProcessorCount * 8, it = 4000;
  thr_kernel<<<blocks, 256>>>(out, 10);
  cudaEventRecord(e0);
  thr_kernel<<<blocks, 256>>>(out, it);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double ops = (double)blocks * 256 * it * 8;
  double per_sm_clk = ops / (ms * 1e-3) / pr.multiProcessorCount / 1.965e9;
  printf("{\"mufu_rsq64h_max_rel_e\": %.3e, \"log2\": %.2f, \"mufu_per_sm_per_clk_at_1965\": %.2f, \"err\": \"%s\"}\n",
         emax, log2(emax), per_sm_clk, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
