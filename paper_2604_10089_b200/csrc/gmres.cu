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
#include <cstdlib>
#include <vector>

#include "bpqn_internal.h"

namespace bpqn {

constexpr int GT = 256;
constexpr int GM_MAX_RESTART = 500;
constexpr int GM_MAX_COEF = 1024;  // coefficient vectors in shared memory: restart or recycle count

// partial dots red[i * nbx + bx] = sum_{e in slice bx} V_i[e] * w[e], i = blockIdx.y
__global__ void k_mdot(const double* __restrict__ V, size_t ld, const double* __restrict__ w, size_t n,
                       double* red, int nbx) {
  const int i = blockIdx.y;
  const double* v = V + (size_t)i * ld;
  double acc = 0.0, acc2 = 0.0;
  if ((n & 1) == 0 && (ld & 1) == 0) {  // 16-byte loads (n = 3N is even for every grid)
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
  } else {
    for (size_t e = (size_t)blockIdx.x * GT + threadIdx.x; e < n; e += (size_t)nbx * GT) acc = fma(v[e], w[e], acc);
  }
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
  __shared__ double sh[GM_MAX_COEF + 1];
  for (int i = threadIdx.x; i < kv; i += blockDim.x) sh[i] = h[i];
  __syncthreads();
  double nrm = 0.0;
  if ((n & 1) == 0 && (ld & 1) == 0) {  // 16-byte loads, two independent chains per thread
    double2* w2 = reinterpret_cast<double2*>(w);
    const size_t n2 = n >> 1, ld2 = ld >> 1;
    const double2* V2 = reinterpret_cast<const double2*>(V);
    for (size_t e = (size_t)blockIdx.x * GT + threadIdx.x; e < n2; e += (size_t)nbx * GT) {
      double2 acc = w2[e];
#pragma unroll 8
      for (int i = 0; i < kv; ++i) {
        const double2 v = V2[(size_t)i * ld2 + e];
        acc.x = fma(-v.x, sh[i], acc.x);
        acc.y = fma(-v.y, sh[i], acc.y);
      }
      w2[e] = acc;
      nrm = fma(acc.x, acc.x, fma(acc.y, acc.y, nrm));
    }
  } else {
    for (size_t e = (size_t)blockIdx.x * GT + threadIdx.x; e < n; e += (size_t)nbx * GT) {
      double acc = w[e];
      for (int i = 0; i < kv; ++i) acc = fma(-V[(size_t)i * ld + e], sh[i], acc);
      w[e] = acc;
      nrm = fma(acc, acc, nrm);
    }
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
constexpr int KD_MAX = 32;  // deflation (GCRO) space dimension cap

struct GmLayout {
  int m;
  size_t H, cs, sn, gv, h1, h2, y, Hraw, Bm, cd, total;
  explicit GmLayout(int mm) : m(mm) {
    H = 8;
    cs = H + (size_t)(m + 1) * m;
    sn = cs + m;
    gv = sn + m;
    h1 = gv + m + 1;
    h2 = h1 + m + 1;
    y = h2 + m + 1;
    Hraw = y + m + 1;                 // unrotated Hessenberg (m+1) x m, column-major
    Bm = Hraw + (size_t)(m + 1) * m;  // B = C^T A V, column k at Bm + k * KD_MAX
    cd = Bm + (size_t)KD_MAX * m;     // KD_MAX coefficients
    total = cd + KD_MAX;
  }
};

// Arnoldi column k: H[:,k] = h1 + h2 (k+1 entries), H[k+1,k] = sqrt(nrm2); apply
// previous rotations, new rotation, update gv; resid = |gv[k+1]| / beta_b.
__global__ void k_givens(double* S, GmLayout L, int k) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double beta_b = S[0];  // |b| (device-resident: the step is replayed as a CUDA graph)
  double* H = S + L.H + (size_t)k * (L.m + 1);
  double* Hr = S + L.Hraw + (size_t)k * (L.m + 1);
  for (int i = 0; i <= k; ++i) Hr[i] = H[i] = S[L.h1 + i] + S[L.h2 + i];
  double bk = sqrt(S[2]);
  S[3] = bk;
  Hr[k + 1] = H[k + 1] = bk;
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
  __shared__ double sy[GM_MAX_COEF + 1];
  for (int i = threadIdx.x; i < kk; i += blockDim.x) sy[i] = y[i];
  __syncthreads();
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
    double acc = x[e];
    for (int i = 0; i < kk; ++i) acc = fma(V[(size_t)i * ld + e], sy[i], acc);
    x[e] = acc;
  }
}

__global__ void k_set(double* d, double v) { *d = v; }

// c[i] = sum_{j<kk} B[j * KD_MAX + i] y[j], i < kd   (GCRO correction B y)
__global__ void k_small_matvec(const double* B, const double* y, int kk, int kd, double* c) {
  const int i = threadIdx.x;
  if (i >= kd) return;
  double acc = 0.0;
  for (int j = 0; j < kk; ++j) acc = fma(B[(size_t)j * KD_MAX + i], y[j], acc);
  c[i] = acc;
}

// out[i][e] = sum_{j<nv} V[j][e] coef[j * nout + i]   (recycle-space construction)
__global__ void k_combine(const double* __restrict__ V, size_t ld, int nv, const double* __restrict__ coef,
                          int nout, double* __restrict__ out, size_t n) {
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
    double acc[KD_MAX];
    for (int i = 0; i < nout; ++i) acc[i] = 0.0;
    for (int j = 0; j < nv; ++j) {
      const double v = V[(size_t)j * ld + e];
      for (int i = 0; i < nout; ++i) acc[i] = fma(v, coef[j * nout + i], acc[i]);
    }
    for (int i = 0; i < nout; ++i) out[(size_t)i * ld + e] = acc[i];
  }
}

// ---- host: small dense linear algebra for the recycle space
// cyclic Jacobi eigen-decomposition of a symmetric n x n matrix (row-major, destroyed);
// eigenvalues in w, eigenvectors as columns of Q (row-major)
static void jacobi_eig(std::vector<double>& A, int n, std::vector<double>& w, std::vector<double>& Q) {
  Q.assign((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i) Q[(size_t)i * n + i] = 1.0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        tot += A[(size_t)i * n + j] * A[(size_t)i * n + j];
        if (i != j) off += A[(size_t)i * n + j] * A[(size_t)i * n + j];
      }
    if (off <= 1e-30 * tot) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = A[(size_t)p * n + q];
        if (std::fabs(apq) < 1e-300) continue;
        const double th = 0.5 * (A[(size_t)q * n + q] - A[(size_t)p * n + p]) / apq;
        const double t = (th >= 0 ? 1.0 : -1.0) / (std::fabs(th) + std::sqrt(th * th + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), sn = t * c;
        for (int k = 0; k < n; ++k) {  // rows p, q
          const double a = A[(size_t)p * n + k], b = A[(size_t)q * n + k];
          A[(size_t)p * n + k] = c * a - sn * b;
          A[(size_t)q * n + k] = sn * a + c * b;
        }
        for (int k = 0; k < n; ++k) {  // columns p, q
          const double a = A[(size_t)k * n + p], b = A[(size_t)k * n + q];
          A[(size_t)k * n + p] = c * a - sn * b;
          A[(size_t)k * n + q] = sn * a + c * b;
        }
        for (int k = 0; k < n; ++k) {
          const double a = Q[(size_t)k * n + p], b = Q[(size_t)k * n + q];
          Q[(size_t)k * n + p] = c * a - sn * b;
          Q[(size_t)k * n + q] = sn * a + c * b;
        }
      }
  }
  w.resize(n);
  for (int i = 0; i < n; ++i) w[i] = A[(size_t)i * n + i];
}

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

// Recycle space for GCRO (R33b): from the last Arnoldi cycle A~ V_kk = V_{kk+1} Hbar
// (A~ = A_op M^-1), the kd right singular vectors G of Hbar with the smallest singular
// values; [Q, R] = qr(Hbar G); C = V_{kk+1} Q (orthonormal), U = V_kk G R^-1, so that
// A~ U = C exactly (no operator applications).  Slow GMRES modes are deflated from
// every later solve on the same operator.
static void build_deflation(Geom& g, const GmLayout& L, int kk, int kd, bool pre, size_t n, cudaStream_t st) {
  kd = std::min(kd, kk - 1);
  if (kd < 1) return;
  std::vector<double> Hr((size_t)(L.m + 1) * kk);
  BPQN_CUDA(cudaMemcpyAsync(Hr.data(), g.scal.p + L.Hraw, Hr.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  BPQN_CUDA(cudaStreamSynchronize(st));
  auto H = [&](int i, int j) { return Hr[(size_t)j * (L.m + 1) + i]; };  // (kk+1) x kk
  std::vector<double> M((size_t)kk * kk, 0.0), w, Q;
  for (int i = 0; i < kk; ++i)
    for (int j = 0; j < kk; ++j) {
      double acc = 0.0;
      for (int r = 0; r <= kk; ++r) acc += H(r, i) * H(r, j);
      M[(size_t)i * kk + j] = acc;
    }
  jacobi_eig(M, kk, w, Q);
  std::vector<int> ord(kk);
  for (int i = 0; i < kk; ++i) ord[i] = i;
  std::sort(ord.begin(), ord.end(), [&](int u, int v) { return w[u] < w[v]; });
  // P = Hbar G, modified Gram-Schmidt twice -> Qp, R
  std::vector<double> G((size_t)kk * kd), P((size_t)(kk + 1) * kd), R((size_t)kd * kd, 0.0);
  for (int c = 0; c < kd; ++c)
    for (int j = 0; j < kk; ++j) G[(size_t)j * kd + c] = Q[(size_t)j * kk + ord[c]];
  for (int r = 0; r <= kk; ++r)
    for (int c = 0; c < kd; ++c) {
      double acc = 0.0;
      for (int j = 0; j < kk; ++j) acc += H(r, j) * G[(size_t)j * kd + c];
      P[(size_t)r * kd + c] = acc;
    }
  double hn = 0.0;
  for (double v : Hr) hn = std::max(hn, std::fabs(v));
  int kept = 0;
  for (int c = 0; c < kd; ++c) {
    for (int pass = 0; pass < 2; ++pass)
      for (int q = 0; q < kept; ++q) {
        double d = 0.0;
        for (int r = 0; r <= kk; ++r) d += P[(size_t)r * kd + q] * P[(size_t)r * kd + c];
        R[(size_t)q * kd + c] += d;
        for (int r = 0; r <= kk; ++r) P[(size_t)r * kd + c] -= d * P[(size_t)r * kd + q];
      }
    double nr = 0.0;
    for (int r = 0; r <= kk; ++r) nr += P[(size_t)r * kd + c] * P[(size_t)r * kd + c];
    nr = std::sqrt(nr);
    if (!(nr > 1e-10 * hn)) break;  // (near) breakdown: stop the space here
    for (int r = 0; r <= kk; ++r) P[(size_t)r * kd + c] /= nr;
    R[(size_t)c * kd + c] = nr;
    if (c != kept) {  // keep columns contiguous
      for (int r = 0; r <= kk; ++r) P[(size_t)r * kd + kept] = P[(size_t)r * kd + c];
      for (int j = 0; j < kk; ++j) G[(size_t)j * kd + kept] = G[(size_t)j * kd + c];
    }
    ++kept;
  }
  if (kept < 1) return;
  kd = kept;
  // Ucoef = G R^-1 (R upper triangular kd x kd, row-major with stride of the original kd)
  const int ks = (int)std::sqrt((double)R.size());
  std::vector<double> Uc((size_t)kk * kd), Cc((size_t)(kk + 1) * kd);
  for (int j = 0; j < kk; ++j)
    for (int c = 0; c < kd; ++c) {  // row j of G times R^-1 by forward substitution
      double acc = G[(size_t)j * ks + c];
      for (int q = 0; q < c; ++q) acc -= Uc[(size_t)j * kd + q] * R[(size_t)q * ks + c];
      Uc[(size_t)j * kd + c] = acc / R[(size_t)c * ks + c];
    }
  for (int r = 0; r <= kk; ++r)
    for (int c = 0; c < kd; ++c) Cc[(size_t)r * kd + c] = P[(size_t)r * ks + c];
  DBuf<double> dUc, dCc;
  dUc.alloc(Uc.size());
  dCc.alloc(Cc.size());
  BPQN_CUDA(cudaMemcpyAsync(dUc.p, Uc.data(), Uc.size() * 8, cudaMemcpyHostToDevice, st));
  BPQN_CUDA(cudaMemcpyAsync(dCc.p, Cc.data(), Cc.size() * 8, cudaMemcpyHostToDevice, st));
  g.def_U.ensure((size_t)KD_MAX * n);
  g.def_C.ensure((size_t)KD_MAX * n);
  const int blocks = std::min<int>((int)((n + 255) / 256), g.sms * 8);
  k_combine<<<blocks, 256, 0, st>>>(g.V.p, n, kk, dUc.p, kd, g.def_U.p, n);
  k_combine<<<blocks, 256, 0, st>>>(g.V.p, n, kk + 1, dCc.p, kd, g.def_C.p, n);
  BPQN_CHECK_LAUNCH();
  BPQN_CUDA(cudaStreamSynchronize(st));
  g.def_k = kd;
  g.def_pre = pre;
}

static bool graphs_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BPQN_GRAPHS");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

static int deflation_dim() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BPQN_DEFLATE");
    v = e ? std::max(0, std::min(KD_MAX, atoi(e))) : 0;  // experimental: off by default
  }
  return v;
}

int gmres_solve(Geom& g, const double* b, double* x, const bpqn_gmres_opts& o, bpqn_gmres_stats& stt,
                cudaStream_t st) {
  const size_t n = 3 * (size_t)g.n;
  const int m = std::max(1, std::min(o.restart, GM_MAX_RESTART));
  const bool pre = o.precond != 0 && g.Minv.p != nullptr;  // block-Jacobi (K4)
  GmLayout L(m);
  g.V.ensure((size_t)(m + 1) * n);
  int nbx = nbx_for(n, g.sms);
  g.red.ensure((size_t)(std::max(m, KD_MAX) + 2) * nbx + 16);
  g.scal.ensure(L.total);
  g.tmp3.ensure(n);
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
  // Recycling (R33): W orthonormal past right-hand sides, Z with
  // A_op Z = W (to the past solves' tolerance).  Initial guess x0 = Z W^T b.  Plus a
  // deflation space (U, C = A~ U) built after the first solve (GCRO, R33b).
  const bool rec = o.recycle != 0 && beta_b > 0.0 && std::isfinite(beta_b);
  if (rec && g.rec_cap == 0) {  // lazily: up to GM_MAX_COEF pairs within ~4 GB (the right-hand sides of
    // LCP MVPs span at most Nc dimensions, so a store of >= Nc pairs ends up predicting them exactly)
    g.rec_cap = (int)std::max<size_t>(1, std::min<size_t>(GM_MAX_COEF, (size_t)4e9 / (2 * n * sizeof(double))));
    g.rec_W.alloc((size_t)g.rec_cap * n);
    g.rec_Z.alloc((size_t)g.rec_cap * n);
    g.rec_k = 0;
    g.def_k = 0;
  }
  const int kr = rec ? g.rec_k : 0;
  const int kd = (rec && g.def_pre == pre) ? g.def_k : 0;  // active deflation dimension
  double* Sc = nullptr;
  if (rec) {
    g.red.ensure((size_t)(std::max(std::max(m, g.rec_cap), KD_MAX) + 2) * nbx + 16);
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
  // x += M^-1 z (or z) for z in tmp3
  auto add_prec = [&](const double* z) {
    if (pre) launch_self_gemm(g, g.Minv.p, z, nullptr, nullptr, x, 1, st);
    else launch_axpby(x, 1.0, z, 1.0, n, st);
  };
  bool first = kr == 0 && kd == 0;
  bool have_x = kr > 0;
  double resid = 1.0;
  int last_kk = 0;
  k_set<<<1, 1, 0, st>>>(S + 0, beta_b);
  // One Arnoldi step (operator, GCRO projection, CGS2, Givens) as device work only: it is
  // captured once per k as a CUDA graph and replayed (launch-bound at small N), unless
  // profiling events, deflation, sharding or BPQN_GRAPHS=0 make it non-capturable.
  auto step_launches = [&](int k, cudaStream_t ss) {
    double* vk = g.V.p + (size_t)k * ld;
    double* w = g.V.p + (size_t)(k + 1) * ld;
    if (pre) {  // right preconditioning: w = A_op M^-1 v_k
      launch_self_gemm(g, g.Minv.p, vk, nullptr, nullptr, g.tmp2.p, 0, ss);
      apply_operator(g, nullptr, g.tmp2.p, nullptr, g.E_A.p, w, ss);
    } else {
      apply_operator(g, nullptr, vk, nullptr, g.E_A.p, w, ss);
    }
    if (kd > 0) {  // (I - C C^T) A~ v_k ; column k of B = C^T A~ v_k
      double* Bk = S + L.Bm + (size_t)k * KD_MAX;
      k_mdot<<<dim3(nbx, kd), GT, 0, ss>>>(g.def_C.p, n, w, n, g.red.p, nbx);
      k_reduce_rows<<<kd, 256, 0, ss>>>(g.red.p, nbx, Bk, 0);
      k_mupdate<<<nbx, GT, 0, ss>>>(g.def_C.p, n, kd, Bk, w, n, nullptr, nbx);
      g.prof.launches += 3;
    }
    // CGS2
    k_mdot<<<dim3(nbx, k + 1), GT, 0, ss>>>(g.V.p, ld, w, n, g.red.p, nbx);
    k_reduce_rows<<<k + 1, 256, 0, ss>>>(g.red.p, nbx, S + L.h1, 0);
    k_mupdate<<<nbx, GT, 0, ss>>>(g.V.p, ld, k + 1, S + L.h1, w, n, nullptr, nbx);
    k_mdot<<<dim3(nbx, k + 1), GT, 0, ss>>>(g.V.p, ld, w, n, g.red.p, nbx);
    k_reduce_rows<<<k + 1, 256, 0, ss>>>(g.red.p, nbx, S + L.h2, 0);
    k_mupdate<<<nbx, GT, 0, ss>>>(g.V.p, ld, k + 1, S + L.h2, w, n, g.red.p, nbx);
    k_reduce_rows<<<1, 256, 0, ss>>>(g.red.p, nbx, S + 2, 0);
    k_givens<<<1, 32, 0, ss>>>(S, L, k);
    k_scale<<<blocks_vec, 256, 0, ss>>>(w, w, n, S + 3, 1);
    BPQN_CHECK_LAUNCH();
    g.prof.launches += 9;
  };
  GraphCache& GC = g.gm_graphs;
  const bool use_graphs = graphs_enabled() && GC.ok && !g.prof.events && kd == 0 && g.shard_world == 1 &&
                          !g.overlap_k2;
  if (use_graphs) GC.validate(g.V.p, g.scal.p, g.red.p, g.tmp2.p, g.packed.p, m, pre);
  auto run_step = [&](int k) {
    if (!use_graphs || !GC.ok) {
      step_launches(k, st);
      return;
    }
    if (!GC.warm[k]) {  // first execution uncaptured (first-use allocations, attribute setup)
      step_launches(k, st);
      GC.warm[k] = 1;
      return;
    }
    if (!GC.exec[k]) {
      if (!GC.cap) BPQN_CUDA(cudaStreamCreateWithFlags(&GC.cap, cudaStreamNonBlocking));
      const long long l0 = g.prof.launches;
      cudaGraph_t graph = nullptr;
      bool ok = cudaStreamBeginCapture(GC.cap, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
      if (ok) {
        try {
          step_launches(k, GC.cap);
        } catch (...) {
          ok = false;
        }
        ok = (cudaStreamEndCapture(GC.cap, &graph) == cudaSuccess) && ok && graph;
      }
      if (ok) ok = cudaGraphInstantiate(&GC.exec[k], graph, 0) == cudaSuccess;
      if (graph) cudaGraphDestroy(graph);
      if (!ok) {  // not capturable here: run uncaptured from now on
        cudaGetLastError();
        GC.ok = false;
        GC.exec[k] = nullptr;
        step_launches(k, st);
        return;
      }
      GC.launches[k] = g.prof.launches - l0;
      g.prof.launches = l0;
    }
    BPQN_CUDA(cudaGraphLaunch(GC.exec[k], st));
    g.prof.launches += GC.launches[k];
  };
  for (;;) {
    double beta;
    if (first) {
      beta = beta_b;
      k_set<<<1, 1, 0, st>>>(S + 3, beta);
      k_scale<<<blocks_vec, 256, 0, st>>>(g.V.p, b, n, S + 3, 1);  // V0 = b / beta
      first = false;
    } else {
      if (have_x) {  // r = b - A x (restart, or the recycled initial guess)
        apply_operator(g, nullptr, x, nullptr, g.E_A.p, g.tmp2.p, st);
        stt.applies++;
        k_sub<<<blocks_vec, 256, 0, st>>>(r, b, g.tmp2.p, n);
        stt.restarts += stt.iters > 0;
      } else {
        BPQN_CUDA(cudaMemcpyAsync(r, b, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
      }
      have_x = true;
      if (kd > 0) {  // GCRO projection: c = C^T r, x += M^-1 U c, r -= C c
        k_mdot<<<dim3(nbx, kd), GT, 0, st>>>(g.def_C.p, n, r, n, g.red.p, nbx);
        k_reduce_rows<<<kd, 256, 0, st>>>(g.red.p, nbx, S + L.cd, 0);
        k_mupdate<<<nbx, GT, 0, st>>>(g.def_C.p, n, kd, S + L.cd, r, n, nullptr, nbx);
        BPQN_CUDA(cudaMemsetAsync(g.tmp3.p, 0, n * sizeof(double), st));
        k_add_basis<<<blocks_vec, 256, 0, st>>>(g.def_U.p, n, kd, S + L.cd, g.tmp3.p, n);
        add_prec(g.tmp3.p);
        BPQN_CHECK_LAUNCH();
        g.prof.launches += 5;
      }
      norm2(g, r, n, S + 2, st);
      beta = std::sqrt(read_scalar(g, S + 2, st));
      if (!(beta > 0.0)) {
        resid = 0.0;
        break;
      }
      resid = beta / beta_b;
      if (!std::isfinite(resid)) {
        status = BPQN_ERR_NAN;
        break;
      }
      if (resid <= o.tol) break;
      k_set<<<1, 1, 0, st>>>(S + 3, beta);
      k_scale<<<blocks_vec, 256, 0, st>>>(g.V.p, r, n, S + 3, 1);
    }
    BPQN_CHECK_LAUNCH();
    k_init_cycle<<<1, 64, 0, st>>>(S, L, beta);
    int kk = 0;
    bool done = false;
    for (int k = 0; k < m; ++k) {
      run_step(k);
      stt.applies++;
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
    // x += M^-1 (V y - U (B y))
    BPQN_CUDA(cudaMemsetAsync(g.tmp3.p, 0, n * sizeof(double), st));
    k_add_basis<<<blocks_vec, 256, 0, st>>>(g.V.p, ld, kk, S + L.y, g.tmp3.p, n);
    if (kd > 0) {
      k_small_matvec<<<1, KD_MAX, 0, st>>>(S + L.Bm, S + L.y, kk, kd, S + L.cd);
      k_mupdate<<<nbx, GT, 0, st>>>(g.def_U.p, n, kd, S + L.cd, g.tmp3.p, n, nullptr, nbx);
      g.prof.launches += 2;
    }
    add_prec(g.tmp3.p);
    BPQN_CHECK_LAUNCH();
    g.prof.launches += 3;
    have_x = true;
    last_kk = kk;
    if (done) break;
  }
  stt.rel_resid = resid;
  // first solve on this operator with recycling: build the deflation space from its last cycle
  const int kdef = deflation_dim();
  if (rec && status == BPQN_OK && g.def_k == 0 && kdef > 0 && last_kk >= kdef + 2)
    build_deflation(g, L, last_kk, kdef, pre, n, st);
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
