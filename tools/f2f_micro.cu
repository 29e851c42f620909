#include <cstdio>
#include <cuda_runtime.h>
// DFMA chains with and without double<->float conversions (which pipe does F2F use on sm_100a?)
template <int MODE>
__global__ void k(double* out, int iters) {
  double a[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) a[c] = 1.0 + 1e-3 * threadIdx.x + c;
  const double m = 0.999999, b = 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      a[c] = fma(a[c], m, b);
      a[c] = fma(a[c], m, b);
      a[c] = fma(a[c], m, b);
      a[c] = fma(a[c], m, b);
      if (MODE == 1) {  // + one double->float->double round trip (2 conversions)
        float f = __double2float_rn(a[c]);
        a[c] += (double)(f * 1e-30f);
      }
      if (MODE == 2) {  // + fp32 MUFU rsqrt seed on a converted value
        float f = __double2float_rn(a[c]);
        float y = rsqrtf(f);
        a[c] = fma((double)y, 1e-30, a[c]);
      }
      if (MODE == 3) {  // + fp64 MUFU.RSQ64H seed
        double y;
        asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a[c]));
        a[c] = fma(y, 1e-30, a[c]);
      }
    }
  }
  double s = 0;
  for (int c = 0; c < 8; ++c) s += a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int MODE>
float run(double* d, int iters) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<MODE><<<148 * 4, 256>>>(d, iters);
  cudaEventRecord(e0);
  k<MODE><<<148 * 4, 256>>>(d, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); return ms;
}
int main() {
  double* d; cudaMalloc(&d, 148 * 4 * 256 * 8);
  int it = 4096;
  float t0 = run<0>(d, it), t1 = run<1>(d, it), t2 = run<2>(d, it), t3 = run<3>(d, it);
  double dfma = 148.0 * 4 * 256 * it * 8 * 4;
  printf("mode0 (4 DFMA)        %.3f ms  %.2f TFLOP/s\n", t0, 2 * dfma / t0 / 1e9);
  printf("mode1 (+F2F round trip + FMUL + DADD) %.3f ms  ratio %.3f\n", t1, t1 / t0);
  printf("mode2 (+F2F + MUFU.RSQ f32 + F2F + DFMA) %.3f ms  ratio %.3f\n", t2, t2 / t0);
  printf("mode3 (+MUFU.RSQ64H + DFMA) %.3f ms  ratio %.3f\n", t3, t3 / t0);
}
