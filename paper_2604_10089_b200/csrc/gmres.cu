// K4: device GMRES for the completed double-layer mobility equation
//   A_op q = rhs,  A_op = -I/2 + D_full + Pi_R     (O7, readings R1-R4, R9)
// Restarted GMRES(m) from q0 = 0 with classical Gram-Schmidt applied twice (CGS2)
// as multi-vector dot-product and update kernels (HBM bound), Givens rotations and
// the residual estimate on the device.  The host only reads one scalar (the
// relative residual) per iteration to decide when to stop.
// Paper: "a traction BIE solve is needed which is done with GMRES until the
// tolerance eps_gmres is met"; the equation itself is reading R1.
#include <algorithm>
#include <cmath>

#include "bpqn_internal.h"

namespace bpqn {

constexpr int GT = 256;
constexpr int GM_MAX_RESTART = 500;

// partial dots red[i * nbx + bx] = sum_{e in slice bx} V_i[e] * w[e], i = blockIdx.y
__global__ void k_mdot(const double* __restrict__ V, size_t ld, const double* __restrict__ w, size_t n,
                       double* red, int nbx) {
  const int i = blockIdx.y;
  const double* v = V + (size_t)i * ld;
  double acc = 0.0;
  for (size_t e = (size_t)blockIdx.x * GT + threadIdx.x; e < n; e += (size_t)nbx * GT) acc = fma(v[e], w[e], acc);
  __shared__ double sred[GT / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double s = threadIdx.x < GT / 32 ? sred[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) red[(size_t)i * nbx + blockIdx.x] = s;
  }
}

// out[i] (+)= sum_bx red[i*nbx + bx], one block per i
__global__ void k_reduce_rows(const double* red, int nbx, double* out, int accumulate) {
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
    if (threadIdx.x == 0) out[i] = accumulate ? out[i] + s : s;
  }
}

// w -= sum_{i<kv} V_i h_i ; red[bx] = partial |w|^2 (if red)
__global__ void k_mupdate(const double* __restrict__ V, size_t ld, int kv, const double* __restrict__ h,
                          double* w, size_t n, double* red, int nbx) {
  __shared__ double sh[GM_MAX_RESTART + 1];
  for (int i = threadIdx.x; i < kv; i += blockDim.x) sh[i] = h[i];
  __syncthreads();
  double nrm = 0.0;
  for (size_t e = (size_t)blockIdx.x * GT + threadIdx.x; e < n; e += (size_t)nbx * GT) {
    double acc = w[e];
    for (int i = 0; i < kv; ++i) acc = fma(-V[(size_t)i * ld + e], sh[i], acc);
    w[e] = acc;
    nrm = fma(acc, acc, nrm);
  }
  if (!red) return;
  __shared__ double sred[GT / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
  if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = nrm;
  __syncthreads();
  if (threadIdx.x < 32) {
    double s = threadIdx.x < GT / 32 ? sred[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) red[blockIdx.x] = s;
  }
}

// y = alpha * x (alpha from device scalar: y = x / sc[0] when inv)
__global__ void k_scale(double* y, const double* x, size_t n, const double* sc, int inv) {
  double a = inv ? (sc[0] > 0.0 ? 1.0 / sc[0] : 0.0) : sc[0];
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x)
    y[e] = a * x[e];
}

// Device GMRES state layout (doubles) inside g.scal:
//   [0] beta0 (|b|)   [1] resid   [2] nrm2 scratch  [3] beta_{k+1}
//   H at 8, (m+1)*m column-major ; cs, sn, gv after ; h1, h2 (m+1 each) ; y (m)
struct GmLayout {
  int m;
  size_t H, cs, sn, gv, h1, h2, y, total;
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

// Arnoldi column k: H[:,k] = h1 + h2 (k+1 entries), H[k+1,k] = sqrt(nrm2); apply
// previous rotations, new rotation, update gv; resid = |gv[k+1]| / beta_b.
__global__ void k_givens(double* S, GmLayout L, int k, double beta_b) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double* H = S + L.H + (size_t)k * (L.m + 1);
  for (int i = 0; i <= k; ++i) H[i] = S[L.h1 + i] + S[L.h2 + i];
  double bk = sqrt(S[2]);
  S[3] = bk;
  H[k + 1] = bk;
  double* cs = S + L.cs;
  double* sn = S + L.sn;
  double* gv = S + L.gv;
  for (int i = 0; i < k; ++i) {
    double t = cs[i] * H[i] + sn[i] * H[i + 1];
    H[i + 1] = -sn[i] * H[i] + cs[i] * H[i + 1];
    H[i] = t;
  }
  double den = hypot(H[k], H[k + 1]);
  double c = den > 0 ? H[k] / den : 1.0, s = den > 0 ? H[k + 1] / den : 0.0;
  cs[k] = c;
  sn[k] = s;
  H[k] = den;
  H[k + 1] = 0.0;
  gv[k + 1] = -s * gv[k];
  gv[k] = c * gv[k];
  S[1] = fabs(gv[k + 1]) / beta_b;
}

// back substitution H[0:kk,0:kk] y = gv[0:kk]
__global__ void k_backsolve(double* S, GmLayout L, int kk) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double* H = S + L.H;
  double* y = S + L.y;
  const double* gv = S + L.gv;
  for (int i = kk - 1; i >= 0; --i) {
    double acc = gv[i];
    for (int j = i + 1; j < kk; ++j) acc -= H[(size_t)j * (L.m + 1) + i] * y[j];
    y[i] = acc / H[(size_t)i * (L.m + 1) + i];
  }
}

__global__ void k_init_cycle(double* S, GmLayout L, double beta) {
  int t = threadIdx.x;
  for (int i = t; i <= L.m; i += blockDim.x) S[L.gv + i] = 0.0;
  if (t == 0) S[L.gv] = beta;
}

// x += V[0:kk] y  (y on device)
__global__ void k_add_basis(const double* __restrict__ V, size_t ld, int kk, const double* y, double* x, size_t n) {
  __shared__ double sy[GM_MAX_RESTART + 1];
  for (int i = threadIdx.x; i < kk; i += blockDim.x) sy[i] = y[i];
  __syncthreads();
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
    double acc = x[e];
    for (int i = 0; i < kk; ++i) acc = fma(V[(size_t)i * ld + e], sy[i], acc);
    x[e] = acc;
  }
}

__global__ void k_set(double* d, double v) { *d = v; }

__global__ void k_sub(double* r, const double* b, const double* ax, size_t n) {
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x)
    r[e] = b[e] - ax[e];
}

static int nbx_for(size_t n, int sms) {
  int nb = (int)std::min<size_t>((n + GT * 4 - 1) / (GT * 4), (size_t)sms * 4);
  return std::max(1, nb);
}

// |v|^2 into S[idx]
static void norm2(Geom& g, const double* v, size_t n, double* dst, cudaStream_t st) {
  int nbx = nbx_for(n, g.sms);
  k_mdot<<<dim3(nbx, 1), GT, 0, st>>>(v, 0, v, n, g.red.p, nbx);
  k_reduce_rows<<<1, 256, 0, st>>>(g.red.p, nbx, dst, 0);
  BPQN_CHECK_LAUNCH();
  g.prof.launches += 2;
}

static double read_scalar(Geom& g, const double* dev, cudaStream_t st) {
  BPQN_CUDA(cudaMemcpyAsync(g.host_scal, dev, sizeof(double), cudaMemcpyDeviceToHost, st));
  BPQN_CUDA(cudaStreamSynchronize(st));
  return g.host_scal[0];
}

int gmres_solve(Geom& g, const double* b, double* x, const bpqn_gmres_opts& o, bpqn_gmres_stats& stt,
                cudaStream_t st) {
  const size_t n = 3 * (size_t)g.n;
  const int m = std::max(1, std::min(o.restart, GM_MAX_RESTART));
  const bool pre = o.precond != 0 && g.Minv.p != nullptr;  // block-Jacobi (K4)
  GmLayout L(m);
  g.V.ensure((size_t)(m + 1) * n);
  int nbx = nbx_for(n, g.sms);
  g.red.ensure((size_t)(m + 2) * nbx + 16);
  g.scal.ensure(L.total);
  double* S = g.scal.p;
  const size_t ld = n;
  cudaEvent_t e0, e1;
  BPQN_CUDA(cudaEventCreate(&e0));
  BPQN_CUDA(cudaEventCreate(&e1));
  BPQN_CUDA(cudaEventRecord(e0, st));

  BPQN_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), st));
  norm2(g, b, n, S + 2, st);
  double beta_b = std::sqrt(read_scalar(g, S + 2, st));
  stt.iters = 0;
  stt.restarts = 0;
  stt.rel_resid = 0.0;
  stt.applies = 0;
  // Recycling: W orthonormal past right-hand sides, Z with
  // A_op Z = W (to the past solves' tolerance).  Initial guess x0 = Z W^T b.
  const bool rec = o.recycle != 0 && beta_b > 0.0 && std::isfinite(beta_b);
  if (rec && g.rec_cap == 0) {  // lazily: up to 256 pairs within ~4 GB
    g.rec_cap = (int)std::max<size_t>(1, std::min<size_t>(256, (size_t)4e9 / (2 * n * sizeof(double))));
    g.rec_W.alloc((size_t)g.rec_cap * n);
    g.rec_Z.alloc((size_t)g.rec_cap * n);
    g.rec_k = 0;
  }
  const int kr = rec ? g.rec_k : 0;
  double* Sc = nullptr;
  if (rec) {
    g.red.ensure((size_t)(std::max(m, g.rec_cap) + 2) * nbx + 16);
    g.scal.ensure(L.total + 2 * (size_t)(g.rec_cap + 1));
    S = g.scal.p;
    Sc = S + L.total;
  }
  if (kr > 0) {
    k_mdot<<<dim3(nbx, kr), GT, 0, st>>>(g.rec_W.p, n, b, n, g.red.p, nbx);
    k_reduce_rows<<<kr, 256, 0, st>>>(g.red.p, nbx, Sc, 0);
    k_add_basis<<<std::min<int>((int)((n + 255) / 256), g.sms * 8), 256, 0, st>>>(g.rec_Z.p, n, kr, Sc, x, n);
    BPQN_CHECK_LAUNCH();
    g.prof.launches += 3;
  }
  int status = BPQN_OK;
  if (!(beta_b > 0.0)) {
    BPQN_CUDA(cudaEventRecord(e1, st));
    BPQN_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    stt.ms = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return std::isfinite(beta_b) ? BPQN_OK : BPQN_ERR_NAN;
  }
  const int blocks_vec = std::min<int>((int)((n + 255) / 256), g.sms * 8);
  double* r = g.tmp.p;
  bool first = kr == 0;
  double resid = 1.0;
  for (;;) {
    double beta;
    if (first) {
      beta = beta_b;
      k_set<<<1, 1, 0, st>>>(S + 3, beta);
      k_scale<<<blocks_vec, 256, 0, st>>>(g.V.p, b, n, S + 3, 1);  // V0 = b / beta
      first = false;
    } else {
      // r = b - A x (restart, or the recycled initial guess)
      apply_operator(g, nullptr, x, nullptr, g.E_A.p, g.tmp2.p, st);
      stt.applies++;
      k_sub<<<blocks_vec, 256, 0, st>>>(r, b, g.tmp2.p, n);
      norm2(g, r, n, S + 2, st);
      beta = std::sqrt(read_scalar(g, S + 2, st));
      if (!(beta > 0.0)) break;
      resid = beta / beta_b;
      if (!std::isfinite(resid)) {
        status = BPQN_ERR_NAN;
        break;
      }
      if (resid <= o.tol) break;
      k_set<<<1, 1, 0, st>>>(S + 3, beta);
      k_scale<<<blocks_vec, 256, 0, st>>>(g.V.p, r, n, S + 3, 1);
      stt.restarts++;
    }
    BPQN_CHECK_LAUNCH();
    k_init_cycle<<<1, 64, 0, st>>>(S, L, beta);
    int kk = 0;
    bool done = false;
    for (int k = 0; k < m; ++k) {
      double* vk = g.V.p + (size_t)k * ld;
      double* w = g.V.p + (size_t)(k + 1) * ld;
      if (pre) {  // right preconditioning: w = A_op M^-1 v_k
        launch_self_gemm(g, g.Minv.p, vk, nullptr, nullptr, g.tmp2.p, 0, st);
        apply_operator(g, nullptr, g.tmp2.p, nullptr, g.E_A.p, w, st);
      } else {
        apply_operator(g, nullptr, vk, nullptr, g.E_A.p, w, st);
      }
      stt.applies++;
      // CGS2
      k_mdot<<<dim3(nbx, k + 1), GT, 0, st>>>(g.V.p, ld, w, n, g.red.p, nbx);
      k_reduce_rows<<<k + 1, 256, 0, st>>>(g.red.p, nbx, S + L.h1, 0);
      k_mupdate<<<nbx, GT, 0, st>>>(g.V.p, ld, k + 1, S + L.h1, w, n, nullptr, nbx);
      k_mdot<<<dim3(nbx, k + 1), GT, 0, st>>>(g.V.p, ld, w, n, g.red.p, nbx);
      k_reduce_rows<<<k + 1, 256, 0, st>>>(g.red.p, nbx, S + L.h2, 0);
      k_mupdate<<<nbx, GT, 0, st>>>(g.V.p, ld, k + 1, S + L.h2, w, n, g.red.p, nbx);
      k_reduce_rows<<<1, 256, 0, st>>>(g.red.p, nbx, S + 2, 0);
      k_givens<<<1, 32, 0, st>>>(S, L, k, beta_b);
      k_scale<<<blocks_vec, 256, 0, st>>>(w, w, n, S + 3, 1);
      BPQN_CHECK_LAUNCH();
      g.prof.launches += 9;
      kk = k + 1;
      stt.iters++;
      resid = read_scalar(g, S + 1, st);
      if (!std::isfinite(resid)) {
        status = BPQN_ERR_NAN;
        done = true;
        break;
      }
      if (resid <= o.tol) {
        done = true;
        break;
      }
      if (stt.iters >= o.max_iters) {
        status = BPQN_ERR_NOCONV;
        done = true;
        break;
      }
    }
    k_backsolve<<<1, 32, 0, st>>>(S, L, kk);
    if (pre) {  // x += M^-1 (V y)
      BPQN_CUDA(cudaMemsetAsync(g.tmp2.p, 0, n * sizeof(double), st));
      k_add_basis<<<blocks_vec, 256, 0, st>>>(g.V.p, ld, kk, S + L.y, g.tmp2.p, n);
      launch_self_gemm(g, g.Minv.p, g.tmp2.p, nullptr, nullptr, x, 1, st);
    } else {
      k_add_basis<<<blocks_vec, 256, 0, st>>>(g.V.p, ld, kk, S + L.y, x, n);
    }
    BPQN_CHECK_LAUNCH();
    g.prof.launches += 2;
    if (done) break;
  }
  stt.rel_resid = resid;
  if (rec && status == BPQN_OK && g.rec_k < g.rec_cap) {
    // append (b, x): CGS2 of b against W with the same coefficients applied to x vs Z
    const size_t ld2 = n;
    double* wn = g.rec_W.p + (size_t)g.rec_k * ld2;
    double* zn = g.rec_Z.p + (size_t)g.rec_k * ld2;
    BPQN_CUDA(cudaMemcpyAsync(wn, b, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    BPQN_CUDA(cudaMemcpyAsync(zn, x, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    const int k0 = g.rec_k;
    for (int pass = 0; pass < 2 && k0 > 0; ++pass) {
      k_mdot<<<dim3(nbx, k0), GT, 0, st>>>(g.rec_W.p, ld2, wn, n, g.red.p, nbx);
      k_reduce_rows<<<k0, 256, 0, st>>>(g.red.p, nbx, Sc, 0);
      k_mupdate<<<nbx, GT, 0, st>>>(g.rec_W.p, ld2, k0, Sc, wn, n, nullptr, nbx);
      k_mupdate<<<nbx, GT, 0, st>>>(g.rec_Z.p, ld2, k0, Sc, zn, n, nullptr, nbx);
      g.prof.launches += 4;
    }
    norm2(g, wn, n, S + 2, st);
    const double nw = std::sqrt(read_scalar(g, S + 2, st));
    if (nw > 1e-8 * beta_b) {  // a new direction: normalise and keep
      k_set<<<1, 1, 0, st>>>(S + 3, nw);
      k_scale<<<blocks_vec, 256, 0, st>>>(wn, wn, n, S + 3, 1);
      k_scale<<<blocks_vec, 256, 0, st>>>(zn, zn, n, S + 3, 1);
      BPQN_CHECK_LAUNCH();
      g.rec_k++;
    }
  }
  BPQN_CUDA(cudaEventRecord(e1, st));
  BPQN_CUDA(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  stt.ms = ms;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return status;
}

}  // namespace bpqn
