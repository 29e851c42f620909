// K4: device GMRES for the completed double-layer mobility equation
//   A_op q = rhs,  A_op = -I/2 + D_full + Pi_R     (O7, readings R1-R4, R9)
// Paper: "a traction BIE solve is needed which is done with GMRES until the tolerance
// eps_gmres is met"; the equation itself is reading R1.
//
// Restarted, right-preconditioned GMRES(m) with classical Gram-Schmidt applied twice (CGS2).
// One Arnoldi step is the operator (K3 preconditioner + K1/K2/K3 layer operator) followed by
// three fused kernels:
//   k_arn_dot      normalise v_k in place, h1 = V^T z                       (last block reduces)
//   k_arn_upd_dot  z -= V h1, h2 = V^T z                                    (last block reduces)
//   k_arn_upd_norm z -= V h2, |z|, u_{k+1} = z; the last block runs the Givens rotations,
//                  the residual estimate and the stopping test, and sets the loop condition
// The operator is applied to the unnormalised u_k = nu_k v_k (so the step needs no separate
// normalisation kernel); the Hessenberg column is divided by nu_k.  Dot products use fixed-
// order block partials (no atomics): the iteration is bit-reproducible.  A whole restart cycle
// runs as ONE CUDA graph whose conditional WHILE node replays the step until the device-side
// test says stop -- the host synchronises once per cycle, not once per iteration.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "bpqn_internal.h"

namespace bpqn {

constexpr int GT = 256;
constexpr int GW = GT / 32;
constexpr int GM_MAX_RESTART = 500;
constexpr int GM_MAX_COEF = 1024;  // coefficient vectors in shared memory: restart or recycle count

// ctl (device ints): [0] k (step in this cycle)  [1] total iterations  [2] NaN flag
//                    [3] continue flag  [4..6] arrival counters of the three fused kernels
// S (device doubles): [0] |b|  [1] resid  [2] |z|^2  [3] nu_k  [4] tol  [5] max iterations
constexpr int GM_CTL = 8;

struct GmLayout {
  int m;
  size_t H, cs, sn, gv, h1, h2, y, total;
  GmLayout() : GmLayout(1) {}
  explicit GmLayout(int mm) : m(mm) {
    H = 8;
    cs = H + (size_t)(m + 1) * m;
    sn = cs + m;
    gv = sn + m;
    h1 = gv + m + 1;
    h2 = h1 + m + 1;
    y = h2 + m + 1;
    total = y + m + 1;
  }
};

// ---------------------------------------------------------------- generic multi-vector kernels
// partial dots red[i * nbx + bx] = sum_{e in slice bx} V_i[e] * w[e], i = blockIdx.y
__global__ void k_mdot(const double* __restrict__ V, size_t ld, const double* __restrict__ w, size_t n,
                       double* red, int nbx) {
  const int i = blockIdx.y;
  const double* v = V + (size_t)i * ld;
  double acc = 0.0, acc2 = 0.0;
  const double2* v2 = reinterpret_cast<const double2*>(v);
  const double2* w2 = reinterpret_cast<const double2*>(w);
  const size_t n2 = n >> 1;
#pragma unroll 4
  for (size_t e = (size_t)blockIdx.x * GT + threadIdx.x; e < n2; e += (size_t)nbx * GT) {
    const double2 a = v2[e], b = w2[e];
    acc = fma(a.x, b.x, acc);
    acc2 = fma(a.y, b.y, acc2);
  }
  acc += acc2;
  __shared__ double sred[GW];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double s = threadIdx.x < GW ? sred[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) red[(size_t)i * nbx + blockIdx.x] = s;
  }
}

// out[i] = sum_bx red[i*nbx + bx], one block per i (fixed order)
__global__ void k_reduce_rows(const double* red, int nbx, double* out) {
  const int i = blockIdx.x;
  double acc = 0.0;
  for (int b = threadIdx.x; b < nbx; b += blockDim.x) acc += red[(size_t)i * nbx + b];
  __shared__ double sred[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double s = threadIdx.x < (int)(blockDim.x / 32) ? sred[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) out[i] = s;
  }
}

// w -= sum_{i<kv} V_i h_i
__global__ void k_mupdate(const double* __restrict__ V, size_t ld, int kv, const double* __restrict__ h, double* w,
                          size_t n) {
  __shared__ double sh[GM_MAX_COEF + 1];
  for (int i = threadIdx.x; i < kv; i += blockDim.x) sh[i] = h[i];
  __syncthreads();
  double2* w2 = reinterpret_cast<double2*>(w);
  const size_t n2 = n >> 1, ld2 = ld >> 1;
  const double2* V2 = reinterpret_cast<const double2*>(V);
  for (size_t e = (size_t)blockIdx.x * GT + threadIdx.x; e < n2; e += (size_t)gridDim.x * GT) {
    double2 acc = w2[e];
#pragma unroll 8
    for (int i = 0; i < kv; ++i) {
      const double2 v = V2[(size_t)i * ld2 + e];
      acc.x = fma(-v.x, sh[i], acc.x);
      acc.y = fma(-v.y, sh[i], acc.y);
    }
    w2[e] = acc;
  }
}

// y = x * a with a = 1 / sc[0] (0 if sc[0] <= 0)
__global__ void k_scale_inv(double* y, const double* x, size_t n, const double* sc) {
  const double a = sc[0] > 0.0 ? 1.0 / sc[0] : 0.0;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x)
    y[e] = a * x[e];
}

// x (+)= sum_{i<kk} V_i y_i, kk = *kkp (device) or kk_host when kkp is null
__global__ void k_add_basis(const double* __restrict__ V, size_t ld, int kk_host, const int* kkp, const double* y,
                            double* x, size_t n, int set) {
  __shared__ double sy[GM_MAX_COEF + 1];
  const int kk = kkp ? *kkp : kk_host;
  for (int i = threadIdx.x; i < kk; i += blockDim.x) sy[i] = y[i];
  __syncthreads();
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
    double acc = set ? 0.0 : x[e];
    for (int i = 0; i < kk; ++i) acc = fma(V[(size_t)i * ld + e], sy[i], acc);
    x[e] = acc;
  }
}

__global__ void k_sub(double* r, const double* b, const double* ax, size_t n) {
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x)
    r[e] = b[e] - ax[e];
}

// ---------------------------------------------------------------- the fused Arnoldi step
// 512 threads per block and 4 independent 16-byte loads in flight per lane: the step's vector work
// is HBM bound (c4: ~4 (k+1) 3N doubles per step), so each SM needs tens of KB of loads in flight.
constexpr int AT = 512;
constexpr int AW = AT / 32;
struct ArnParams {
  double* V;          // basis [(m+1)][ld]
  size_t ld, n;       // n = 3N (even)
  double* z;          // operator output (fixed buffer)
  double* vin;        // operator input u_{k+1} (fixed buffer)
  double* red;        // [(m+2)][nbx] block partials
  int nbx, chunk2;    // blocks, double2 elements per block slice
  int* ctl;
  double* S;
  GmLayout L;
  cudaGraphConditionalHandle cond;
  int use_cond;
};

// this block's slice [e0, e1) in double2 units
__device__ __forceinline__ void arn_slice(const ArnParams& P, size_t& e0, size_t& e1) {
  e0 = (size_t)blockIdx.x * P.chunk2;
  e1 = min(P.n >> 1, e0 + (size_t)P.chunk2);
}

// partial dots of rows 0..k with the slice of z (warp per row, 4 loads in flight per lane),
// red[i * nbx + bx]
__device__ __forceinline__ void arn_block_dots(const ArnParams& P, int k, size_t e0, size_t e1) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double2* z2 = reinterpret_cast<const double2*>(P.z);
  for (int i = warp; i <= k; i += AW) {
    const double2* v2 = reinterpret_cast<const double2*>(P.V + (size_t)i * P.ld);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    size_t e = e0 + lane;
    for (; e + 96 < e1; e += 128) {
      const double2 v0 = v2[e], v1 = v2[e + 32], v2_ = v2[e + 64], v3 = v2[e + 96];
      const double2 w0 = z2[e], w1 = z2[e + 32], w2 = z2[e + 64], w3 = z2[e + 96];
      a0 = fma(v0.x, w0.x, fma(v0.y, w0.y, a0));
      a1 = fma(v1.x, w1.x, fma(v1.y, w1.y, a1));
      a2 = fma(v2_.x, w2.x, fma(v2_.y, w2.y, a2));
      a3 = fma(v3.x, w3.x, fma(v3.y, w3.y, a3));
    }
    for (; e < e1; e += 32) {
      const double2 v = v2[e], w = z2[e];
      a0 = fma(v.x, w.x, fma(v.y, w.y, a0));
    }
    a0 = (a0 + a1) + (a2 + a3);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a0 += __shfl_xor_sync(0xffffffffu, a0, o);
    if (lane == 0) P.red[(size_t)i * P.nbx + blockIdx.x] = a0;
  }
}

// last block to arrive (counter ctl[c]) sums the partials of rows 0..rows-1 into out (fixed order)
__device__ __forceinline__ bool arn_last_block(const ArnParams& P, int c) {
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(P.ctl + c, 1) == P.nbx - 1;
  __syncthreads();
  if (s_last) {
    __threadfence();
    if (threadIdx.x == 0) P.ctl[c] = 0;
  }
  return s_last != 0;
}

__device__ __forceinline__ void arn_sum_rows(const ArnParams& P, int rows, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = warp; i < rows; i += AW) {
    double a = 0.0;
    for (int b = lane; b < P.nbx; b += 32) a += __ldcg(P.red + (size_t)i * P.nbx + b);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) out[i] = a;
  }
}

// z -= sum_{i<=k} V_i h_i on the slice (rows in groups of 4: 4 loads in flight per thread);
// optionally copy the result to dst1/dst2 and return |z|^2 of this thread's elements
__device__ __forceinline__ double arn_block_update(const ArnParams& P, int k, const double* h, size_t e0, size_t e1,
                                                   double* dst1, double* dst2) {
  __shared__ double sh[GM_MAX_RESTART + 1];
  for (int i = threadIdx.x; i <= k; i += blockDim.x) sh[i] = h[i];
  __syncthreads();
  double2* z2 = reinterpret_cast<double2*>(P.z);
  const size_t ld2 = P.ld >> 1;
  const double2* V2 = reinterpret_cast<const double2*>(P.V);
  double nrm = 0.0;
  for (size_t e = e0 + threadIdx.x; e < e1; e += AT) {
    double2 acc = z2[e];
    int i = 0;
    for (; i + 3 <= k; i += 4) {
      const double2 v0 = V2[(size_t)i * ld2 + e], v1 = V2[(size_t)(i + 1) * ld2 + e];
      const double2 v2 = V2[(size_t)(i + 2) * ld2 + e], v3 = V2[(size_t)(i + 3) * ld2 + e];
      acc.x = fma(-v0.x, sh[i], acc.x);
      acc.y = fma(-v0.y, sh[i], acc.y);
      acc.x = fma(-v1.x, sh[i + 1], acc.x);
      acc.y = fma(-v1.y, sh[i + 1], acc.y);
      acc.x = fma(-v2.x, sh[i + 2], acc.x);
      acc.y = fma(-v2.y, sh[i + 2], acc.y);
      acc.x = fma(-v3.x, sh[i + 3], acc.x);
      acc.y = fma(-v3.y, sh[i + 3], acc.y);
    }
    for (; i <= k; ++i) {
      const double2 v = V2[(size_t)i * ld2 + e];
      acc.x = fma(-v.x, sh[i], acc.x);
      acc.y = fma(-v.y, sh[i], acc.y);
    }
    z2[e] = acc;
    if (dst1) reinterpret_cast<double2*>(dst1)[e] = acc;
    if (dst2) reinterpret_cast<double2*>(dst2)[e] = acc;
    nrm = fma(acc.x, acc.x, fma(acc.y, acc.y, nrm));
  }
  return nrm;
}

// (1) v_k = u_k / nu_k in place; h1 = V_{0..k}^T z
__global__ void __launch_bounds__(AT) k_arn_dot(ArnParams P) {
  const int k = P.ctl[0];
  size_t e0, e1;
  arn_slice(P, e0, e1);
  {
    const double nu = P.S[3];
    const double inv = nu > 0.0 ? 1.0 / nu : 0.0;
    double2* vk = reinterpret_cast<double2*>(P.V + (size_t)k * P.ld);
    for (size_t e = e0 + threadIdx.x; e < e1; e += AT) {
      double2 v = vk[e];
      v.x *= inv;
      v.y *= inv;
      vk[e] = v;
    }
  }
  __syncthreads();
  arn_block_dots(P, k, e0, e1);
  if (arn_last_block(P, 4)) arn_sum_rows(P, k + 1, P.S + P.L.h1);
}

// (2) z -= V h1; h2 = V^T z
__global__ void __launch_bounds__(AT) k_arn_upd_dot(ArnParams P) {
  const int k = P.ctl[0];
  size_t e0, e1;
  arn_slice(P, e0, e1);
  arn_block_update(P, k, P.S + P.L.h1, e0, e1, nullptr, nullptr);
  __syncthreads();
  arn_block_dots(P, k, e0, e1);
  if (arn_last_block(P, 5)) arn_sum_rows(P, k + 1, P.S + P.L.h2);
}

// (3) z -= V h2; u_{k+1} = z into V_{k+1} and the operator input; |z|; Givens; stopping test
__global__ void __launch_bounds__(AT) k_arn_upd_norm(ArnParams P) {
  const int k = P.ctl[0];
  size_t e0, e1;
  arn_slice(P, e0, e1);
  double nrm = arn_block_update(P, k, P.S + P.L.h2, e0, e1, P.V + (size_t)(k + 1) * P.ld, P.vin);
  __shared__ double sred[AW];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
  if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = nrm;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < AW; ++w) s += sred[w];
    P.red[blockIdx.x] = s;
  }
  if (!arn_last_block(P, 6)) return;
  if (threadIdx.x >= 32) return;
  {
    double a = 0.0;
    for (int b = threadIdx.x; b < P.nbx; b += 32) a += __ldcg(P.red + b);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (threadIdx.x) return;
    P.S[2] = a;
  }
  double* S = P.S;
  const GmLayout& L = P.L;
  const double nu_k = S[3], nu_n = sqrt(S[2]);
  const double sc = nu_k > 0.0 ? 1.0 / nu_k : 0.0;
  double* H = S + L.H + (size_t)k * (L.m + 1);
  for (int i = 0; i <= k; ++i) H[i] = (S[L.h1 + i] + S[L.h2 + i]) * sc;
  H[k + 1] = nu_n * sc;
  double* cs = S + L.cs;
  double* sn = S + L.sn;
  double* gv = S + L.gv;
  for (int i = 0; i < k; ++i) {
    const double t = cs[i] * H[i] + sn[i] * H[i + 1];
    H[i + 1] = -sn[i] * H[i] + cs[i] * H[i + 1];
    H[i] = t;
  }
  const double den = hypot(H[k], H[k + 1]);
  const double c = den > 0 ? H[k] / den : 1.0, s = den > 0 ? H[k + 1] / den : 0.0;
  cs[k] = c;
  sn[k] = s;
  H[k] = den;
  H[k + 1] = 0.0;
  gv[k + 1] = -s * gv[k];
  gv[k] = c * gv[k];
  const double resid = fabs(gv[k + 1]) / S[0];
  S[1] = resid;
  S[3] = nu_n;
  const int kn = k + 1, it = P.ctl[1] + 1;
  P.ctl[0] = kn;
  P.ctl[1] = it;
  const bool bad = !(resid == resid) || !isfinite(resid) || !(den == den);
  if (bad) P.ctl[2] = 1;
  const int cont = (!bad && resid > S[4] && kn < L.m && (double)it < S[5]) ? 1 : 0;
  P.ctl[3] = cont;
  if (P.use_cond) cudaGraphSetConditional(P.cond, cont);
}

// cycle start: V_0 = u_0 = src, operator input = src, nu_0 = beta, gv = beta e_1, k = 0
__global__ void k_cycle_init(const double* src, double* V0, double* vin, size_t n, double* S, GmLayout L, int* ctl,
                             double beta, int iters) {
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
    const double v = src[e];
    V0[e] = v;
    vin[e] = v;
  }
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i <= L.m; i += blockDim.x) S[L.gv + i] = 0.0;
    if (threadIdx.x == 0) {
      S[L.gv] = beta;
      S[3] = beta;
      ctl[0] = 0;
      ctl[1] = iters;
      ctl[2] = 0;
      ctl[3] = 1;
    }
  }
}

// back substitution H[0:kk,0:kk] y = gv[0:kk], kk = ctl[0]: column-oriented, one block; after y_i
// is known every thread updates its rows j < i in parallel (kk barrier steps instead of a serial
// kk^2/2 chain of dependent global loads)
__global__ void k_backsolve(double* S, GmLayout L, const int* ctl) {
  __shared__ double r[GM_MAX_RESTART + 1];
  __shared__ double yi;
  const int kk = ctl[0];
  const double* H = S + L.H;
  for (int j = threadIdx.x; j < kk; j += blockDim.x) r[j] = S[L.gv + j];
  __syncthreads();
  for (int i = kk - 1; i >= 0; --i) {
    if (threadIdx.x == 0) {
      yi = r[i] / H[(size_t)i * (L.m + 1) + i];
      S[L.y + i] = yi;
    }
    __syncthreads();
    const double* col = H + (size_t)i * (L.m + 1);
    for (int j = threadIdx.x; j < i; j += blockDim.x) r[j] -= col[j] * yi;
    __syncthreads();
  }
}

__global__ void k_set(double* d, double v) { *d = v; }
__global__ void k_set2(double* d, double a, double b) {
  d[0] = a;
  d[1] = b;
}

// ---------------------------------------------------------------- host helpers
static int nbx_for(size_t n, int sms) {
  int nb = (int)std::min<size_t>((n + GT * 4 - 1) / (GT * 4), (size_t)sms * 4);
  return std::max(1, nb);
}

// |v|^2 into dst (device)
static void norm2(Geom& g, const double* v, size_t n, double* dst, cudaStream_t st) {
  int nbx = nbx_for(n, g.sms);
  k_mdot<<<dim3(nbx, 1), GT, 0, st>>>(v, 0, v, n, g.red.p, nbx);
  k_reduce_rows<<<1, 256, 0, st>>>(g.red.p, nbx, dst);
  BPQN_CHECK_LAUNCH();
  g.prof.launches += 2;
}

static double read_scalar(Geom& g, const double* dev, cudaStream_t st) {
  BPQN_CUDA(cudaMemcpyAsync(g.host_scal, dev, sizeof(double), cudaMemcpyDeviceToHost, st));
  BPQN_CUDA(cudaStreamSynchronize(st));
  return g.host_scal[0];
}

static bool graphs_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BPQN_GRAPHS");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// Workspace for restart length m (allocated at geometry init for the default m; a larger m
// requested by a caller is allocated on that call).
void gmres_reserve(Geom& g, int m) {
  const size_t n = 3 * (size_t)g.n;
  m = std::max(1, std::min(m, GM_MAX_RESTART));
  const int nbx = std::max(nbx_for(n, g.sms), 2 * g.sms);
  g.V.ensure((size_t)(m + 1) * n);
  g.red.ensure((size_t)(std::max(m, 1) + 2) * nbx + 16);
  g.scal.ensure(GmLayout(m).total + 2 * (size_t)(GM_MAX_COEF + 1));
  g.gm_ctl.ensure(GM_CTL);
  g.tmp3.ensure(n);
  g.gm_z.ensure(n);
  g.gm_vin.ensure(n);
  if (!g.gm_ctl_init) {
    BPQN_CUDA(cudaMemset(g.gm_ctl.p, 0, sizeof(int) * GM_CTL));
    g.gm_ctl_init = true;
  }
}

// Recycling store (R33): up to GM_MAX_COEF pairs, within ~4 GB and a quarter of the free device
// memory.  Allocated here, outside the hot calls; on failure recycling stays off (rec_cap = 0).
void gmres_recycle_reserve(Geom& g) {
  if (g.rec_cap > 0) return;
  const size_t n = 3 * (size_t)g.n;
  size_t fr = 0, tot = 0;
  if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) fr = (size_t)8e9;
  const size_t budget = std::min<size_t>((size_t)4e9, fr / 4);
  const int cap = (int)std::min<size_t>(GM_MAX_COEF, budget / (2 * n * sizeof(double)));
  if (cap < 1) return;
  double *W = nullptr, *Z = nullptr;
  if (cudaMalloc(&W, (size_t)cap * n * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&Z, (size_t)cap * n * sizeof(double)) != cudaSuccess) {
    cudaGetLastError();
    if (W) cudaFree(W);
    return;  // recycle stays off
  }
  g.rec_W.release();
  g.rec_Z.release();
  g.rec_W.p = W;
  g.rec_W.n = (size_t)cap * n;
  g.rec_Z.p = Z;
  g.rec_Z.n = (size_t)cap * n;
  g.rec_cap = cap;
  g.rec_k = 0;
  g.red.ensure((size_t)(cap + 2) * nbx_for(n, g.sms) + 16);  // recycle dots: cap rows of block partials
  g.gm_cycle.clear();  // the captured cycle holds the old red address
}

// ---------------------------------------------------------------- the solver
int gmres_solve(Geom& g, const double* b, double* x, const bpqn_gmres_opts& o, bpqn_gmres_stats& stt,
                cudaStream_t st) {
  const size_t n = 3 * (size_t)g.n;
  BPQN_REQUIRE((n & 1) == 0, "3N must be even");
  const int m = std::max(1, std::min(o.restart, GM_MAX_RESTART));
  const bool pre = o.precond != 0 && g.Minv.p != nullptr;  // block-Jacobi (K4)
  GmLayout L(m);
  // FMM-accelerated refinement (bpqn_gmres_opts.relax_fmm): every Krylov step applies the operator with
  // the FMM far field; each cycle reduces its own residual by relax_delta and the next one starts from the
  // DIRECT residual b - A x, which alone decides convergence (defect correction with an approximate inner
  // operator: the error contracts by ~|I - A A_fmm^-1| + delta per cycle)
  const bool relax = o.relax_fmm != 0;
  BPQN_REQUIRE(!relax || g.fmm, "relax_fmm needs a handle built with fmm_order > 0");
  const double relax_delta = o.relax_delta > 0.0 ? std::min(o.relax_delta, 0.5) : 3e-3;
  double cycle_tol = o.tol;
  FmmDirect direct(g, relax);  // direct applications outside the Krylov steps
  gmres_reserve(g, m);  // no-op unless this restart length exceeds the reserved one
  const int nbx_v = nbx_for(n, g.sms);
  double* S = g.scal.p;
  double* Sc = S + L.total;  // recycling coefficients
  int* ctl = g.gm_ctl.p;
  const size_t ld = n;
  cudaEvent_t e0, e1;
  BPQN_CUDA(cudaEventCreate(&e0));
  BPQN_CUDA(cudaEventCreate(&e1));
  BPQN_CUDA(cudaEventRecord(e0, st));
  auto finish = [&](int status) {
    BPQN_CUDA(cudaEventRecord(e1, st));
    BPQN_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    stt.ms = ms;
    if (!relax && g.fmm && g.fmm_on) stt.fmm_applies = stt.applies;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return status;
  };

  BPQN_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), st));
  norm2(g, b, n, S + 2, st);
  const double beta_b = std::sqrt(read_scalar(g, S + 2, st));
  stt.iters = 0;
  stt.restarts = 0;
  stt.rel_resid = 0.0;
  stt.applies = 0;
  stt.fmm_applies = 0;
  if (!(beta_b > 0.0)) return finish(std::isfinite(beta_b) ? BPQN_OK : BPQN_ERR_NAN);
  // Recycling (R33): W orthonormal past right-hand sides, Z with
  // A_op Z = W (to the past solves' tolerance).  Initial guess x0 = Z W^T b.  Needs a store
  // reserved outside the hot call (bpqn_gmres_recycle_reset / bpqn_solve_lcp); else off.
  const bool rec = o.recycle != 0 && g.rec_cap > 0;
  const int kr = rec ? g.rec_k : 0;
  if (kr > 0) {
    k_mdot<<<dim3(nbx_v, kr), GT, 0, st>>>(g.rec_W.p, n, b, n, g.red.p, nbx_v);
    k_reduce_rows<<<kr, 256, 0, st>>>(g.red.p, nbx_v, Sc);
    k_add_basis<<<std::min<int>((int)((n + 255) / 256), g.sms * 8), 256, 0, st>>>(g.rec_Z.p, n, kr, nullptr, Sc,
                                                                                  x, n, 0);
    BPQN_CHECK_LAUNCH();
    g.prof.launches += 3;
  }
  const int blocks_vec = std::min<int>((int)((n + 255) / 256), g.sms * 8);
  k_set2<<<1, 1, 0, st>>>(S + 4, o.tol, (double)o.max_iters);
  k_set<<<1, 1, 0, st>>>(S + 0, beta_b);
  BPQN_CHECK_LAUNCH();

  // the fused step's launch geometry: one slice per block, nbx blocks covering n/2 double2
  ArnParams A;
  A.V = g.V.p;
  A.ld = ld;
  A.n = n;
  A.z = g.gm_z.p;
  A.vin = g.gm_vin.p;
  A.red = g.red.p;
  // up to 2 blocks per SM, slices of >= 64 double2: small systems (c1, p_lo = 4) still fill the GPU
  A.nbx = std::max(1, std::min<int>(2 * g.sms, (int)((n / 2 + 63) / 64)));
  A.chunk2 = (int)((n / 2 + A.nbx - 1) / A.nbx);
  A.ctl = ctl;
  A.S = S;
  A.L = L;
  A.cond = 0;
  A.use_cond = 0;
  auto step_launches = [&](cudaStream_t ss, const ArnParams& P) {
    if (pre) {  // right preconditioning: z = A_op M^-1 u_k
      launch_self_gemm(g, g.Minv.p, g.gm_vin.p, g.tmp2.p, 0, ss);
      apply_operator(g, nullptr, g.tmp2.p, nullptr, g.E_A.p, g.gm_z.p, ss);
    } else {
      apply_operator(g, nullptr, g.gm_vin.p, nullptr, g.E_A.p, g.gm_z.p, ss);
    }
    k_arn_dot<<<P.nbx, AT, 0, ss>>>(P);
    k_arn_upd_dot<<<P.nbx, AT, 0, ss>>>(P);
    k_arn_upd_norm<<<P.nbx, AT, 0, ss>>>(P);
    BPQN_CHECK_LAUNCH();
    g.prof.launches += 3;
  };

  // one restart cycle as a CUDA graph: a conditional WHILE node around the step (built once per
  // handle and restart length; not when profiling events, sharding or BPQN_GRAPHS=0 make the step
  // non-capturable)
  CycleGraph& CG = g.gm_cycle;
  // callback sharding synchronises the stream inside the operator (not capturable); the NCCL sharding
  // enqueues its collectives on the streams and is captured like the single-GPU step (falls back to
  // host-driven steps if the capture or instantiation is refused)
  const bool capturable_shard = !g.sharded() || (g.nccl_comm && !g.sh_fn && !g.sh_rs_fn);
  const bool use_graphs =
      graphs_enabled() && !g.prof.events && capturable_shard && !g.overlap_k2 && CG.ok;
  if (CG.exec && (CG.m != m || CG.pre != pre || CG.V != g.V.p || CG.S != g.scal.p || CG.red != g.red.p))
    CG.clear();
  auto build_graph = [&]() -> bool {
    if (!CG.cap) BPQN_CUDA(cudaStreamCreateWithFlags(&CG.cap, cudaStreamNonBlocking));
    bool ok = cudaGraphCreate(&CG.graph, 0) == cudaSuccess;
    ok = ok && cudaGraphConditionalHandleCreate(&CG.h, CG.graph, 1, cudaGraphCondAssignDefault) == cudaSuccess;
    cudaGraphNode_t node;
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = CG.h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    ok = ok && cudaGraphAddNode(&node, CG.graph, nullptr, 0, &cp) == cudaSuccess;
    if (ok) {
      cudaGraph_t body = cp.conditional.phGraph_out[0];
      ArnParams P = A;
      P.cond = CG.h;
      P.use_cond = 1;
      const long long l0 = g.prof.launches, a0 = g.prof.allpairs_launches;
      ok = cudaStreamBeginCaptureToGraph(CG.cap, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) ==
           cudaSuccess;
      if (ok) {
        try {
          step_launches(CG.cap, P);
        } catch (...) {
          ok = false;
        }
        cudaGraph_t out = nullptr;
        ok = (cudaStreamEndCapture(CG.cap, &out) == cudaSuccess) && ok;
      }
      CG.launches = g.prof.launches - l0;
      CG.k1 = g.prof.allpairs_launches - a0;
      g.prof.launches = l0;
      g.prof.allpairs_launches = a0;
    }
    ok = ok && cudaGraphInstantiate(&CG.exec, CG.graph, 0) == cudaSuccess;
    if (!ok) {
      cudaGetLastError();
      CG.clear();
      CG.ok = false;  // not capturable here: host-driven steps from now on
      if (getenv("BPQN_LOG_MVP")) fprintf(stderr, "gmres: cycle graph not capturable, host-driven steps\n");
      return false;
    }
    CG.m = m;
    CG.pre = pre;
    CG.V = g.V.p;
    CG.S = g.scal.p;
    CG.red = g.red.p;
    return true;
  };

  double* r = g.tmp.p;
  bool first = true;
  double resid = 1.0;
  int status = BPQN_OK;
  for (;;) {
    double beta;
    const double* src;
    if (first && kr == 0) {
      beta = beta_b;
      src = b;
    } else {  // r = b - A x (restart, or the recycled initial guess)
      apply_operator(g, nullptr, x, nullptr, g.E_A.p, g.tmp2.p, st);
      stt.applies++;
      k_sub<<<blocks_vec, 256, 0, st>>>(r, b, g.tmp2.p, n);
      stt.restarts += stt.iters > 0;
      norm2(g, r, n, S + 2, st);
      beta = std::sqrt(read_scalar(g, S + 2, st));
      src = r;
      if (!(beta > 0.0)) {
        resid = 0.0;
        break;
      }
      resid = beta / beta_b;
      if (!std::isfinite(resid)) {
        status = BPQN_ERR_NAN;
        break;
      }
      if (relax && getenv("BPQN_LOG_MVP")) fprintf(stderr, "fmm refinement: direct residual %.3e\n", resid);
      if (resid <= o.tol) break;
    }
    first = false;
    if (relax) {  // this cycle's target: its own residual reduced by relax_delta (never below tol)
      cycle_tol = std::max(o.tol, relax_delta * beta / beta_b);
      k_set<<<1, 1, 0, st>>>(S + 4, cycle_tol);
    }
    k_cycle_init<<<blocks_vec, 256, 0, st>>>(src, g.V.p, g.gm_vin.p, n, S, L, ctl, beta, stt.iters);
    BPQN_CHECK_LAUNCH();
    g.prof.launches++;
    if (stt.iters >= o.max_iters) {
      status = BPQN_ERR_NOCONV;
      break;
    }
    // steps of this cycle (FMM refinement: with the FMM far field -- the same graph as a plain FMM handle's)
    if (relax) g.fmm_on = true;
    bool graphed = false;
    if (use_graphs && CG.ok) {
      if (!CG.exec && CG.warm) build_graph();
      if (CG.exec) {
        BPQN_CUDA(cudaGraphLaunch(CG.exec, st));
        graphed = true;
      }
    }
    int h[4];
    if (!graphed) {  // host-driven: one step, then read the device's stopping decision
      for (int k = 0; k < m; ++k) {
        step_launches(st, A);
        BPQN_CUDA(cudaMemcpyAsync(h, ctl, 4 * sizeof(int), cudaMemcpyDeviceToHost, st));
        BPQN_CUDA(cudaStreamSynchronize(st));
        if (!h[3]) break;
      }
      CG.warm = true;  // first use done uncaptured (attribute setup, occupancy queries)
    }
    if (relax) g.fmm_on = false;
    BPQN_CUDA(cudaMemcpyAsync(h, ctl, 4 * sizeof(int), cudaMemcpyDeviceToHost, st));
    BPQN_CUDA(cudaMemcpyAsync(g.host_scal, S + 1, sizeof(double), cudaMemcpyDeviceToHost, st));
    BPQN_CUDA(cudaStreamSynchronize(st));
    const int kk = h[0];
    if (graphed) {
      g.prof.launches += CG.launches * kk;
      g.prof.allpairs_launches += CG.k1 * kk;
    }
    stt.applies += kk;
    if (relax) stt.fmm_applies += kk;
    stt.iters = h[1];
    resid = g.host_scal[0];
    bool done = false;
    if (h[2] || !std::isfinite(resid)) {
      status = BPQN_ERR_NAN;
      done = true;
    } else if (resid <= cycle_tol) {
      // FMM refinement: the estimate belongs to the FMM operator -- the next pass of the loop forms the
      // direct residual b - A x and stops only if that meets tol
      done = !relax;
    } else if (stt.iters >= o.max_iters) {
      status = BPQN_ERR_NOCONV;
      done = true;
    }
    if (kk > 0) {  // x += M^-1 V y
      k_backsolve<<<1, 128, 0, st>>>(S, L, ctl);
      k_add_basis<<<blocks_vec, 256, 0, st>>>(g.V.p, ld, 0, ctl, S + L.y, g.tmp3.p, n, 1);
      BPQN_CHECK_LAUNCH();
      if (pre) launch_self_gemm(g, g.Minv.p, g.tmp3.p, x, 1, st);
      else launch_axpby(x, 1.0, g.tmp3.p, 1.0, n, st);
      g.prof.launches += 2;
    }
    if (done) break;
  }
  stt.rel_resid = resid;
  if (rec && status == BPQN_OK && g.rec_k < g.rec_cap) {
    // append (b, x): CGS2 of b against W with the same coefficients applied to x vs Z
    double* wn = g.rec_W.p + (size_t)g.rec_k * n;
    double* zn = g.rec_Z.p + (size_t)g.rec_k * n;
    BPQN_CUDA(cudaMemcpyAsync(wn, b, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    BPQN_CUDA(cudaMemcpyAsync(zn, x, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    const int k0 = g.rec_k;
    for (int pass = 0; pass < 2 && k0 > 0; ++pass) {
      k_mdot<<<dim3(nbx_v, k0), GT, 0, st>>>(g.rec_W.p, n, wn, n, g.red.p, nbx_v);
      k_reduce_rows<<<k0, 256, 0, st>>>(g.red.p, nbx_v, Sc);
      k_mupdate<<<nbx_v, GT, 0, st>>>(g.rec_W.p, n, k0, Sc, wn, n);
      k_mupdate<<<nbx_v, GT, 0, st>>>(g.rec_Z.p, n, k0, Sc, zn, n);
      g.prof.launches += 4;
    }
    norm2(g, wn, n, S + 2, st);
    const double nw = std::sqrt(read_scalar(g, S + 2, st));
    // keep any new direction above 1e-8 |b|.  The stored z = (x - Z c) / nw carries x's error
    // (~tol |b|) divided by nw, so nearly dependent directions are less accurate; a tol-tied
    // threshold max(1e-8, sqrt(tol)) |b| was measured to cost more than it saves (c4 Bi-PQN:
    // 16 045 -> 19 440 lo GMRES iterations): initial guesses only need to be good, the true
    // residual decides convergence.
    if (nw > 1e-8 * beta_b) {
      k_set<<<1, 1, 0, st>>>(S + 2, nw);
      k_scale_inv<<<blocks_vec, 256, 0, st>>>(wn, wn, n, S + 2);
      k_scale_inv<<<blocks_vec, 256, 0, st>>>(zn, zn, n, S + 2);
      BPQN_CHECK_LAUNCH();
      g.rec_k++;
    }
  }
  return finish(status);
}

}  // namespace bpqn
