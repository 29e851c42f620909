// FP64 peak microbenchmarks for B200 (sm_100a): DFMA pipe, DMMA (mma.sync f64),
// and the MUFU.RSQ64H-seeded rsqrt sequence. Writes one JSON line to stdout.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define NCHAIN 8
__global__ void dfma_kernel(double* out, double a, double b, int iters) {
  double x[NCHAIN];
#pragma unroll
  for (int c = 0; c < NCHAIN; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int c = 0; c < NCHAIN; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < NCHAIN; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, b0 = 1.0 - threadIdx.x * 1e-4;
  double d[4][2];
#pragma unroll
  for (int c = 0; c < 4; ++c) d[c][0] = d[c][1] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int c = 0; c < 4; ++c)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a0), "d"(b0));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) s += d[c][0] + d[c][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void rsqrt_kernel(double* out, int iters) {
  double x[NCHAIN], acc[NCHAIN];
#pragma unroll
  for (int c = 0; c < NCHAIN; ++c) { x[c] = 1.0 + threadIdx.x * 1e-3 + c; acc[c] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < NCHAIN; ++c) { acc[c] += rsqrt(x[c]); x[c] += 1e-9; }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < NCHAIN; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

// DFMA chains and DMMA issued by the same warps: if the two shared one pipe the time would be
// the sum of the pure kernels' times; if they are separate units it approaches the max.
__global__ void mix_kernel(double* out, double a, double b, int iters) {
  double x[NCHAIN];
#pragma unroll
  for (int c = 0; c < NCHAIN; ++c) x[c] = threadIdx.x * 1e-3 + c;
  double a0 = threadIdx.x * 1e-3, b0 = 1.0 - threadIdx.x * 1e-4;
  double d[4][2];
#pragma unroll
  for (int c = 0; c < 4; ++c) d[c][0] = d[c][1] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int c = 0; c < NCHAIN; ++c) x[c] = fma(x[c], a, b);
#pragma unroll
      for (int c = 0; c < 4; ++c)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a0), "d"(b0));
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < NCHAIN; ++c) s += x[c];
#pragma unroll
  for (int c = 0; c < 4; ++c) s += d[c][0] + d[c][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int dev = 0; cudaDeviceProp pr; cudaGetDeviceProperties(&pr, dev);
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  double* out; cudaMalloc(&out, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = pr.multiProcessorCount;
  int blocks = sms * 8, threads = 256;
  float ms;
  // DFMA
  int it = 4000;
  dfma_kernel<<<blocks, threads>>>(out, 0.999999, 1e-7, 10);
  cudaEventRecord(e0); dfma_kernel<<<blocks, threads>>>(out, 0.999999, 1e-7, it); cudaEventRecord(e1);
  cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  double dfma_tf = 2.0 * blocks * threads * (double)it * 16 * NCHAIN / (ms * 1e-3) / 1e12;
  // DMMA m8n8k4: 2*8*8*4 = 512 flop per warp-instruction
  int it2 = 2000;
  dmma_kernel<<<blocks, threads>>>(out, 10);
  cudaEventRecord(e0); dmma_kernel<<<blocks, threads>>>(out, it2); cudaEventRecord(e1);
  cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  double dmma_tf = 512.0 * (blocks * threads / 32) * (double)it2 * 8 * 4 / (ms * 1e-3) / 1e12;
  // rsqrt
  int it3 = 4000;
  rsqrt_kernel<<<blocks, threads>>>(out, 10);
  cudaEventRecord(e0); rsqrt_kernel<<<blocks, threads>>>(out, it3); cudaEventRecord(e1);
  cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  double rsqrt_g = (double)blocks * threads * it3 * NCHAIN / (ms * 1e-3) / 1e9;
  // mixed: per iteration 8 x NCHAIN DFMA (as dfma_kernel at half the unroll) + 8 x 4 DMMA (as dmma_kernel)
  int it4 = 2000;
  mix_kernel<<<blocks, threads>>>(out, 0.999999, 1e-7, 10);
  cudaEventRecord(e0); mix_kernel<<<blocks, threads>>>(out, 0.999999, 1e-7, it4); cudaEventRecord(e1);
  cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  double mix_ms = ms;
  double mix_dfma_tf = 2.0 * blocks * threads * (double)it4 * 8 * NCHAIN / (ms * 1e-3) / 1e12;
  double mix_dmma_tf = 512.0 * (blocks * threads / 32) * (double)it4 * 8 * 4 / (ms * 1e-3) / 1e12;
  // the same work done by the pure kernels back to back would take t_dfma + t_dmma
  double t_sep = 2.0 * blocks * threads * (double)it4 * 8 * NCHAIN / (dfma_tf * 1e12) * 1e3 +
                 512.0 * (blocks * threads / 32) * (double)it4 * 8 * 4 / (dmma_tf * 1e12) * 1e3;
  printf("{\"mix_ms\": %.3f, \"sum_of_pure_ms\": %.3f, \"mix_dfma_tflops\": %.3f, \"mix_dmma_tflops\": %.3f}\n",
         mix_ms, t_sep, mix_dfma_tf, mix_dmma_tf);
  cudaError_t err = cudaGetLastError();
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_attr_mhz\": %.0f, \"dfma_tflops\": %.3f, \"dmma_m8n8k4_tflops\": %.3f, \"rsqrt_f64_gops\": %.2f, \"err\": \"%s\"}\n",
         pr.name, sms, clk_khz / 1e3, dfma_tf, dmma_tf, rsqrt_g, cudaGetErrorString(err));
  return 0;
}
