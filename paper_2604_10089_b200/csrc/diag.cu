// Diagnostics of libbpqn (not on the hot path): an exhaustive check of the MUFU.RSQ64H seed bound
// that K1 / K2 rely on (allpairs.cu header: rho^-k = y^k (1 - e)^(-k/2) truncated after e^2, with
// e = 1 - rho^2 y^2 and |e| <= 2^-19 so that the truncation error is < 7 |e|^3 ~ 4e-17).
#include <cstdint>
#include <cstring>

#include "bpqn_internal.h"

namespace bpqn {

// One thread per (exponent, 20-bit high mantissa) pattern of rr: the seed instruction reads the
// high word, so over the 2^32 low-word values e = 1 - rr y^2 is monotone in rr and its extremes are
// at low word 0 and 0xffffffff.  max |e| is accumulated as the bit pattern of a positive double
// (integer order = value order).
__global__ void k_rsq_sweep(int e_lo, int n_exp, unsigned long long* max_bits) {
  const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (long long)n_exp << 20) return;
  const int ex = e_lo + (int)(id >> 20);
  const unsigned mant = (unsigned)(id & 0xfffff);
  const unsigned hi = ((unsigned)(ex + 1023) << 20) | mant;
  double worst = 0.0;
  for (int k = 0; k < 2; ++k) {
    const double rr = __hiloint2double((int)hi, k ? (int)0xffffffffu : 0);
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(rr));
    const double e = fma(-rr, y * y, 1.0);
    worst = fmax(worst, fabs(e));
  }
  atomicMax(max_bits, (unsigned long long)__double_as_longlong(worst));
}

}  // namespace bpqn

using namespace bpqn;

extern "C" int bpqn_diag_rsqrt_seed(int exp_lo, int exp_hi, double* max_abs_e) {
  try {
    BPQN_REQUIRE(max_abs_e && exp_hi >= exp_lo && exp_lo >= -1022 && exp_hi <= 1023, "bad arguments");
    unsigned long long* d = nullptr;
    BPQN_CUDA(cudaMalloc(&d, sizeof(unsigned long long)));
    BPQN_CUDA(cudaMemset(d, 0, sizeof(unsigned long long)));
    const int n_exp = exp_hi - exp_lo + 1;
    const long long n = (long long)n_exp << 20;
    k_rsq_sweep<<<(unsigned)((n + 255) / 256), 256>>>(exp_lo, n_exp, d);
    BPQN_CUDA(cudaGetLastError());
    unsigned long long h = 0;
    BPQN_CUDA(cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost));
    cudaFree(d);
    double v;
    static_assert(sizeof(v) == sizeof(h), "");
    memcpy(&v, &h, sizeof(v));
    *max_abs_e = v;
    return BPQN_OK;
  } catch (const Error& e) {
    set_error(e.msg);
    return e.code;
  }
}
