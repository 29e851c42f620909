// H1: host-side Mono-PQN / Bi-PQN (the paper's outer loop) for libbpqn.
//
// Alg. 1 Mono-PQN, Alg. 2 optimal over-relaxation
// (P:372-388), Alg. 3 Bi-PQN, Prop. 1 / Alg. 4 weighted prox via
// semi-smooth Newton, unrolled full-memory BFGS (App. D.1
// P:802-810), cached low-fidelity secant (App. D.2).  Readings R11
// (x~ = x - tau H g), R15 (prox residual with the +[a; a~] term), R16-R19, R22.
//
// Runs on the host (OpenMP for the O(Nc r^2) and O(r^3) prox pieces): one Nc-vector
// crosses PCIe per MVP.  C^{-1} = (D + UU^T)^{-1} is applied by the Woodbury identity.
#include <algorithm>
#include <chrono>
#include <immintrin.h>
#include <omp.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <functional>
#include <limits>
#include <stdexcept>
#include <vector>

#include "pqn.h"

namespace bpqn {

using Vec = std::vector<double>;

static double dot(const Vec& a, const Vec& b) {
  double s = 0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}
static double nrm(const Vec& a) { return std::sqrt(dot(a, a)); }

// dense LU solve (partial pivoting) of a small system; returns false if singular
static bool lu_solve(std::vector<double> A, int n, Vec& b) {
  std::vector<int> piv(n);
  for (int k = 0; k < n; ++k) {
    int pm = k;
    for (int i = k + 1; i < n; ++i)
      if (std::fabs(A[i * n + k]) > std::fabs(A[pm * n + k])) pm = i;
    if (A[pm * n + k] == 0.0) return false;
    if (pm != k) {
      for (int j = 0; j < n; ++j) std::swap(A[k * n + j], A[pm * n + j]);
      std::swap(b[k], b[pm]);
    }
    for (int i = k + 1; i < n; ++i) {
      double f = A[i * n + k] / A[k * n + k];
      for (int j = k; j < n; ++j) A[i * n + j] -= f * A[k * n + j];
      b[i] -= f * b[k];
    }
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = b[i];
    for (int j = i + 1; j < n; ++j) s -= A[i * n + j] * b[j];
    b[i] = s / A[i * n + i];
  }
  return true;
}

double kkt_abs(const Vec& x, const Vec& g) {
  double s = 0;
  for (size_t i = 0; i < x.size(); ++i) {
    double m = std::min(x[i], g[i]);
    s += m * m;
  }
  return std::sqrt(s);
}

// ------------------------------------------------------------------ BFGS
void Bfgs::clear() {
  U.clear();
  V.clear();
  S.clear();
  Y.clear();
  wc = WoodburyCache();
}
Vec Bfgs::B(const Vec& x) const {
  Vec out = x;
  for (auto& u : U) {
    double c = dot(u, x);
    for (size_t i = 0; i < out.size(); ++i) out[i] += c * u[i];
  }
  for (auto& v : V) {
    double c = dot(v, x);
    for (size_t i = 0; i < out.size(); ++i) out[i] -= c * v[i];
  }
  return out;
}
Vec Bfgs::H(const Vec& g) const {
  Vec q = g;
  std::vector<double> al(S.size());
  for (int k = (int)S.size() - 1; k >= 0; --k) {
    double rho = 1.0 / dot(Y[k], S[k]);
    al[k] = rho * dot(S[k], q);
    for (size_t i = 0; i < q.size(); ++i) q[i] -= al[k] * Y[k][i];
  }
  for (size_t k = 0; k < S.size(); ++k) {
    double rho = 1.0 / dot(Y[k], S[k]);
    double be = rho * dot(Y[k], q);
    for (size_t i = 0; i < q.size(); ++i) q[i] += S[k][i] * (al[k] - be);
  }
  return q;
}
bool Bfgs::update(const Vec& s, const Vec& y, const Vec* Bs_in, double curv) {
  double ys = dot(y, s);
  if (!std::isfinite(ys)) throw std::runtime_error("NaN in BFGS update");
  if (ys <= curv * nrm(s) * nrm(y)) return false;
  Vec Bs = Bs_in ? *Bs_in : B(s);
  double sBs = dot(s, Bs);
  if (!(sBs > 0)) return false;
  Vec u(s.size()), v(s.size());
  double a = 1.0 / std::sqrt(ys), b = 1.0 / std::sqrt(sBs);
  for (size_t i = 0; i < s.size(); ++i) {
    u[i] = a * y[i];
    v[i] = b * Bs[i];
  }
  U.push_back(u);
  V.push_back(v);
  S.push_back(s);
  Y.push_back(y);
  return true;
}

// ------------------------------------------------------------------ dense kernels (host)
// Row-major small dense linear algebra for the prox; OpenMP over rows once the
// problem is big enough to pay (Bi-PQN seeds the subproblem memory with every
// earlier secant pair, so r reaches a few hundred, "full memory").
static bool par(long long work) { return work > 200000; }

// C[m x n] (ldc) += sign A[m x k] (lda) B[k x n] (ldb), row-major.  AVX2 micro-kernel: 4 rows x 8 columns of
// C in 8 ymm accumulators, per k two B loads and four broadcasts of A; scalar edges; OpenMP over 4-row
// blocks (each C element has one owner: deterministic).
static void mk_gemm(double* C, int ldc, const double* A, int lda, const double* B, int ldb, int m, int n, int k,
                    bool subtract) {
  const int m4 = m / 4 * 4, n8 = n / 8 * 8;
  const double sg = subtract ? -1.0 : 1.0;
#pragma omp parallel for schedule(static) if ((long long)m * n * k > 4000000)  // fork/join pays only here
  for (int i = 0; i < m4; i += 4) {
    const double* l0 = A + (size_t)i * lda;
    const double* l1 = l0 + lda;
    const double* l2 = l1 + lda;
    const double* l3 = l2 + lda;
    for (int j = 0; j < n8; j += 8) {
      double* c0 = C + (size_t)i * ldc + j;
      __m256d a00 = _mm256_loadu_pd(c0), a01 = _mm256_loadu_pd(c0 + 4);
      __m256d a10 = _mm256_loadu_pd(c0 + ldc), a11 = _mm256_loadu_pd(c0 + ldc + 4);
      __m256d a20 = _mm256_loadu_pd(c0 + 2 * ldc), a21 = _mm256_loadu_pd(c0 + 2 * ldc + 4);
      __m256d a30 = _mm256_loadu_pd(c0 + 3 * ldc), a31 = _mm256_loadu_pd(c0 + 3 * ldc + 4);
      const double* u = B + j;
      if (subtract) {
        for (int kk = 0; kk < k; ++kk, u += ldb) {
          const __m256d u0 = _mm256_loadu_pd(u), u1 = _mm256_loadu_pd(u + 4);
          __m256d t = _mm256_broadcast_sd(l0 + kk);
          a00 = _mm256_fnmadd_pd(t, u0, a00); a01 = _mm256_fnmadd_pd(t, u1, a01);
          t = _mm256_broadcast_sd(l1 + kk);
          a10 = _mm256_fnmadd_pd(t, u0, a10); a11 = _mm256_fnmadd_pd(t, u1, a11);
          t = _mm256_broadcast_sd(l2 + kk);
          a20 = _mm256_fnmadd_pd(t, u0, a20); a21 = _mm256_fnmadd_pd(t, u1, a21);
          t = _mm256_broadcast_sd(l3 + kk);
          a30 = _mm256_fnmadd_pd(t, u0, a30); a31 = _mm256_fnmadd_pd(t, u1, a31);
        }
      } else {
        for (int kk = 0; kk < k; ++kk, u += ldb) {
          const __m256d u0 = _mm256_loadu_pd(u), u1 = _mm256_loadu_pd(u + 4);
          __m256d t = _mm256_broadcast_sd(l0 + kk);
          a00 = _mm256_fmadd_pd(t, u0, a00); a01 = _mm256_fmadd_pd(t, u1, a01);
          t = _mm256_broadcast_sd(l1 + kk);
          a10 = _mm256_fmadd_pd(t, u0, a10); a11 = _mm256_fmadd_pd(t, u1, a11);
          t = _mm256_broadcast_sd(l2 + kk);
          a20 = _mm256_fmadd_pd(t, u0, a20); a21 = _mm256_fmadd_pd(t, u1, a21);
          t = _mm256_broadcast_sd(l3 + kk);
          a30 = _mm256_fmadd_pd(t, u0, a30); a31 = _mm256_fmadd_pd(t, u1, a31);
        }
      }
      _mm256_storeu_pd(c0, a00); _mm256_storeu_pd(c0 + 4, a01);
      _mm256_storeu_pd(c0 + ldc, a10); _mm256_storeu_pd(c0 + ldc + 4, a11);
      _mm256_storeu_pd(c0 + 2 * ldc, a20); _mm256_storeu_pd(c0 + 2 * ldc + 4, a21);
      _mm256_storeu_pd(c0 + 3 * ldc, a30); _mm256_storeu_pd(c0 + 3 * ldc + 4, a31);
    }
    for (int r = 0; r < 4; ++r)
      for (int j = n8; j < n; ++j) {
        double acc = 0.0;
        for (int kk = 0; kk < k; ++kk) acc += A[(size_t)(i + r) * lda + kk] * B[(size_t)kk * ldb + j];
        C[(size_t)(i + r) * ldc + j] += sg * acc;
      }
  }
  for (int i = m4; i < m; ++i)
    for (int j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int kk = 0; kk < k; ++kk) acc += A[(size_t)i * lda + kk] * B[(size_t)kk * ldb + j];
      C[(size_t)i * ldc + j] += sg * acc;
    }
}

// C[m x p] = A[m x k] B[p x k]^T (+ C if acc): B transposed once, then the micro-kernel GEMM
static void gemm_nt(const double* A, const double* B, double* C, int m, int p, int k, bool acc) {
  std::vector<double> Bt((size_t)k * p);
  for (int j = 0; j < p; ++j)
    for (int e = 0; e < k; ++e) Bt[(size_t)e * p + j] = B[(size_t)j * k + e];
  if (!acc) std::fill(C, C + (size_t)m * p, 0.0);
  mk_gemm(C, p, A, k, Bt.data(), p, m, p, k, false);
}

// in-place Cholesky K = L L^T (lower), false if not positive definite
static bool cholesky(std::vector<double>& K, int n) {
  for (int j = 0; j < n; ++j) {
    double d = K[(size_t)j * n + j];
    for (int k = 0; k < j; ++k) d -= K[(size_t)j * n + k] * K[(size_t)j * n + k];
    if (!(d > 0.0)) return false;
    d = std::sqrt(d);
    K[(size_t)j * n + j] = d;
#pragma omp parallel for schedule(static) if (par((long long)(n - j) * j))
    for (int i = j + 1; i < n; ++i) {
      double s = K[(size_t)i * n + j];
      for (int k = 0; k < j; ++k) s -= K[(size_t)i * n + k] * K[(size_t)j * n + k];
      K[(size_t)i * n + j] = s / d;
    }
  }
  return true;
}

// X[n x m] (row-major, columns are right-hand sides) <- K^{-1} X with K = L L^T
static void chol_solve(const std::vector<double>& L, int n, double* X, int m) {
#pragma omp parallel for schedule(static) if (par((long long)n * n * m))
  for (int c = 0; c < m; ++c) {
    for (int i = 0; i < n; ++i) {
      double s = X[(size_t)i * m + c];
      for (int k = 0; k < i; ++k) s -= L[(size_t)i * n + k] * X[(size_t)k * m + c];
      X[(size_t)i * m + c] = s / L[(size_t)i * n + i];
    }
    for (int i = n - 1; i >= 0; --i) {
      double s = X[(size_t)i * m + c];
      for (int k = i + 1; k < n; ++k) s -= L[(size_t)k * n + i] * X[(size_t)k * m + c];
      X[(size_t)i * m + c] = s / L[(size_t)i * n + i];
    }
  }
}

// LU with partial pivoting, one right-hand side.  One OpenMP team for the whole
// factorisation (no fork/join per column): the pivot search and swap run on one thread,
// the trailing update is split by rows; the solve is serial.
static bool lu_solve_par(std::vector<double>& A, int n, Vec& b) {
  bool ok = true;
  const int nt = par((long long)n * n * n / 3) ? 0 : 1;  // 0: default team size
#pragma omp parallel num_threads(nt > 0 ? nt : omp_get_max_threads())
  {
    for (int k = 0; k < n; ++k) {
#pragma omp single
      {
        int pm = k;
        for (int i = k + 1; i < n; ++i)
          if (std::fabs(A[(size_t)i * n + k]) > std::fabs(A[(size_t)pm * n + k])) pm = i;
        if (A[(size_t)pm * n + k] == 0.0) {
          ok = false;
        } else if (pm != k) {
          for (int j = 0; j < n; ++j) std::swap(A[(size_t)k * n + j], A[(size_t)pm * n + j]);
          std::swap(b[k], b[pm]);
        }
      }  // implicit barrier
      if (!ok) break;
      const double piv = A[(size_t)k * n + k];
      const double* rk = &A[(size_t)k * n];
#pragma omp for schedule(static)
      for (int i = k + 1; i < n; ++i) {
        double* ri = &A[(size_t)i * n];
        const double f = ri[k] / piv;
        if (f == 0.0) continue;
#pragma omp simd
        for (int j = k; j < n; ++j) ri[j] -= f * rk[j];
        b[i] -= f * b[k];
      }  // implicit barrier
    }
  }
  if (!ok) return false;
  for (int i = n - 1; i >= 0; --i) {
    double s = b[i];
    for (int j = i + 1; j < n; ++j) s -= A[(size_t)i * n + j] * b[j];
    b[i] = s / A[(size_t)i * n + i];
  }
  return true;
}

// Blocked right-looking LU with partial pivoting (panel width 32) and one right-hand side: the
// panel is factored by one thread, the U12 block row and the trailing update A22 -= L21 U12 run
// in an OpenMP team with the column loop vectorised (the rank-1-per-column version spent 1.19 s
// of a c4 Bi-PQN solve in 564 factorisations of mean order 371).
static bool lu_solve_blocked(std::vector<double>& A, int n, Vec& b) {
  constexpr int NB = 32;
  if (n <= 2 * NB) return lu_solve_par(A, n, b);
  std::vector<int> piv(n);
  bool ok = true;
  for (int k0 = 0; k0 < n && ok; k0 += NB) {
    const int kb = std::min(NB, n - k0), k1 = k0 + kb;
    for (int k = k0; k < k1; ++k) {  // panel (rows k..n-1, columns k..k1-1)
      int pm = k;
      for (int i = k + 1; i < n; ++i)
        if (std::fabs(A[(size_t)i * n + k]) > std::fabs(A[(size_t)pm * n + k])) pm = i;
      piv[k] = pm;
      if (A[(size_t)pm * n + k] == 0.0) {
        ok = false;
        break;
      }
      if (pm != k)
        for (int j = 0; j < n; ++j) std::swap(A[(size_t)k * n + j], A[(size_t)pm * n + j]);
      const double inv = 1.0 / A[(size_t)k * n + k];
      const double* rk = &A[(size_t)k * n];
      for (int i = k + 1; i < n; ++i) {
        double* ri = &A[(size_t)i * n];
        const double f = (ri[k] *= inv);
        if (f != 0.0)
          for (int j = k + 1; j < k1; ++j) ri[j] -= f * rk[j];
      }
    }
    if (!ok || k1 >= n) break;
    // U12 = L11^-1 A12 (unit lower) and A22 -= L21 U12
#pragma omp parallel
    {
#pragma omp for schedule(static)
      for (int jb = k1; jb < n; jb += 64) {
        const int je = std::min(n, jb + 64);
        for (int k = k0; k < k1; ++k)
          for (int i = k + 1; i < k1; ++i) {
            const double f = A[(size_t)i * n + k];
            double* ri = &A[(size_t)i * n];
            const double* rk = &A[(size_t)k * n];
#pragma omp simd
            for (int j = jb; j < je; ++j) ri[j] -= f * rk[j];
          }
      }
    }
    // trailing update A22 -= L21 U12 in place (micro-kernel GEMM, row blocks over the OpenMP team)
    const int m = n - k1;
    mk_gemm(&A[(size_t)k1 * n + k1], n, &A[(size_t)k1 * n + k0], n, &A[(size_t)k0 * n + k1], n, m, m, kb, true);
  }
  if (!ok) return false;
  for (int k = 0; k < n; ++k)
    if (piv[k] != k) std::swap(b[k], b[piv[k]]);
  for (int i = 1; i < n; ++i) {  // unit lower
    double s = b[i];
    const double* ri = &A[(size_t)i * n];
    for (int j = 0; j < i; ++j) s -= ri[j] * b[j];
    b[i] = s;
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = b[i];
    const double* ri = &A[(size_t)i * n];
    for (int j = i + 1; j < n; ++j) s -= ri[j] * b[j];
    b[i] = s / ri[i];
  }
  return true;
}

// ------------------------------------------------------------------ weighted prox
// prox^B_{x>=0}(x~), B = I + UU^T - VV^T (D = I in both solvers, R19), by the dual
// root of Prop. 1 with Alg. 4's semi-smooth Newton on the
// residual with the "+[alpha; alpha~]" term restored (R15).  C^{-1} V by Woodbury
// with one Cholesky factor of I + U^T U; the Jacobian blocks of P:709-712 as
// products over the active / inactive coordinates.
struct ProxTimers {
  double setup = 0, jac = 0, lu = 0, resid = 0;
  long calls = 0, newton = 0, rsum = 0;
  ~ProxTimers() {
    if (getenv("BPQN_PQN_PROFILE"))
      fprintf(stderr, "prox: calls %ld newton %ld avg r %.1f | setup %.3fs jac %.3fs lu %.3fs resid %.3fs\n", calls,
              newton, calls ? (double)rsum / calls : 0.0, setup, jac, lu, resid);
  }
};
static thread_local ProxTimers g_pt;  // per solving thread (handles are single-owner)
void prox_profile_flush() {  // BPQN_PQN_PROFILE: report and reset (called after each solve)
  if (!getenv("BPQN_PQN_PROFILE")) return;
  fprintf(stderr, "prox: calls %ld newton %ld avg r %.1f | setup %.3fs jac %.3fs lu %.3fs resid %.3fs\n", g_pt.calls,
          g_pt.newton, g_pt.calls ? (double)g_pt.rsum / g_pt.calls : 0.0, g_pt.setup, g_pt.jac, g_pt.lu, g_pt.resid);
  g_pt.setup = g_pt.jac = g_pt.lu = g_pt.resid = 0;
  g_pt.calls = g_pt.newton = g_pt.rsum = 0;
}
static double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// Bring q.wc up to date with q.U / q.V (see WoodburyCache).  Full build: CU = U K^-1,
// CV = V - U K^-1 U^T V with K = I + U^T U (Cholesky); append of (u, v): w = C^-1 u,
// den = 1 + u.w, CU_i -= w (w.U_i)/den, CV_i -= w (w.V_i)/den, then CU_new = w/den,
// CV_new = C^-1 v - w (w.v)/den with C^-1 x = x - sum_i CU_i (U_i.x) of the old memory.
static void woodbury_update(const Bfgs& q, int n) {
  WoodburyCache& W = q.wc;
  const int r = (int)q.U.size();
  const bool full = W.n != n || W.r > r || W.appends + (r - W.r) > 64 || W.r == 0 ||
                    (r > 0 && W.r > 0 && !std::equal(q.U[W.r - 1].begin(), q.U[W.r - 1].end(),
                                                     W.Um.begin() + (size_t)(W.r - 1) * n));
  if (full) {
    W = WoodburyCache();
    W.n = n;
    W.r = r;
    W.Um.resize((size_t)r * n);
    W.Vm.resize((size_t)r * n);
    W.CU.resize((size_t)r * n);
    W.CV.resize((size_t)r * n);
    for (int c = 0; c < r; ++c) {
      std::copy(q.U[c].begin(), q.U[c].end(), W.Um.begin() + (size_t)c * n);
      std::copy(q.V[c].begin(), q.V[c].end(), W.Vm.begin() + (size_t)c * n);
    }
    if (r == 0) return;
    // K = I + U^T U; X = K^-1 [U^T U | U^T V]; CU_c = U_c - sum_i X[i][c] U_i ... written as
    // CU = U K^-1 (columns c: sum_i U_i Kinv[i][c]) and CV = V - U K^-1 U^T V
    std::vector<double> K((size_t)r * r), X((size_t)r * 2 * r, 0.0), G((size_t)r * r);
    gemm_nt(W.Um.data(), W.Um.data(), K.data(), r, r, n, false);
    for (int i = 0; i < r; ++i) K[(size_t)i * r + i] += 1.0;
    if (!cholesky(K, r)) throw std::runtime_error("Woodbury core not positive definite");
    gemm_nt(W.Um.data(), W.Vm.data(), G.data(), r, r, n, false);  // G[i][c] = U_i . V_c
    for (int i = 0; i < r; ++i) {
      X[(size_t)i * 2 * r + i] = 1.0;  // identity -> K^-1
      for (int c = 0; c < r; ++c) X[(size_t)i * 2 * r + r + c] = G[(size_t)i * r + c];
    }
    chol_solve(K, r, X.data(), 2 * r);
#pragma omp parallel for schedule(static) if (par((long long)r * r * n))
    for (int c = 0; c < r; ++c) {
      double* ou = &W.CU[(size_t)c * n];
      double* ov = &W.CV[(size_t)c * n];
      std::fill(ou, ou + n, 0.0);
      std::copy(&W.Vm[(size_t)c * n], &W.Vm[(size_t)c * n] + n, ov);
      for (int i = 0; i < r; ++i) {
        const double fu = X[(size_t)i * 2 * r + c], fv = X[(size_t)i * 2 * r + r + c];
        const double* u = &W.Um[(size_t)i * n];
#pragma omp simd
        for (int e = 0; e < n; ++e) {
          ou[e] += fu * u[e];
          ov[e] -= fv * u[e];
        }
      }
    }
    return;
  }
  for (int k = W.r; k < r; ++k) {  // append pair k
    const Vec& u = q.U[k];
    const Vec& v = q.V[k];
    const int r0 = W.r;
    // w = C^-1 u, z = C^-1 v with the current (old) memory
    Vec cu(r0), cv(r0);
#pragma omp parallel for schedule(static) if (par((long long)r0 * n * 2))
    for (int i = 0; i < r0; ++i) {
      const double* Ui = &W.Um[(size_t)i * n];
      double su = 0.0, sv = 0.0;
      for (int e = 0; e < n; ++e) {
        su += Ui[e] * u[e];
        sv += Ui[e] * v[e];
      }
      cu[i] = su;
      cv[i] = sv;
    }
    Vec w = u, z = v;
    for (int i = 0; i < r0; ++i) {
      const double* Ci = &W.CU[(size_t)i * n];
      for (int e = 0; e < n; ++e) {
        w[e] -= Ci[e] * cu[i];
        z[e] -= Ci[e] * cv[i];
      }
    }
    const double den = 1.0 + dot(u, w);
    // rank-one correction of the existing columns
#pragma omp parallel for schedule(static) if (par((long long)r0 * n * 2))
    for (int i = 0; i < r0; ++i) {
      double* ci = &W.CU[(size_t)i * n];
      double* vi = &W.CV[(size_t)i * n];
      const double* Ui = &W.Um[(size_t)i * n];
      const double* Vi = &W.Vm[(size_t)i * n];
      double a = 0.0, b = 0.0;
      for (int e = 0; e < n; ++e) {
        a += w[e] * Ui[e];
        b += w[e] * Vi[e];
      }
      a /= den;
      b /= den;
      for (int e = 0; e < n; ++e) {
        ci[e] -= a * w[e];
        vi[e] -= b * w[e];
      }
    }
    const double wv = dot(w, v) / den;
    W.Um.insert(W.Um.end(), u.begin(), u.end());
    W.Vm.insert(W.Vm.end(), v.begin(), v.end());
    for (int e = 0; e < n; ++e) W.CU.push_back(w[e] / den);
    for (int e = 0; e < n; ++e) W.CV.push_back(z[e] - wv * w[e]);
    W.r = k + 1;
    W.appends++;
  }
}

Vec weighted_prox(const Bfgs& q, const Vec& xt, double tol, int jmax, int* iters) {
  const int n = (int)xt.size();
  const int r = (int)q.U.size();
  g_pt.calls++;
  g_pt.rsum += r;
  double t_0 = now_s();
  if (r == 0) {
    Vec z(n);
    for (int i = 0; i < n; ++i) z[i] = std::max(xt[i], 0.0);
    if (iters) *iters = 0;
    return z;
  }
  if (tol <= 0) {
    double mx = 1.0;
    for (double v : xt) mx = std::max(mx, std::fabs(v));
    tol = 1e-12 * mx;
  }
  woodbury_update(q, n);
  const std::vector<double>& Um = q.wc.Um;
  const std::vector<double>& Vm = q.wc.Vm;
  const std::vector<double>& CV = q.wc.CV;
  const int d = 2 * r;
  g_pt.setup += now_s() - t_0;
  auto residual = [&](const Vec& a, Vec& L, Vec& z, std::vector<char>& act) {
    Vec y = xt, v(n);
    for (int c = 0; c < r; ++c) {
      const double* cv = &CV[(size_t)c * n];
      const double ac = a[r + c];
      for (int e = 0; e < n; ++e) y[e] += cv[e] * ac;
    }
    v = y;
    for (int c = 0; c < r; ++c) {
      const double* u = &Um[(size_t)c * n];
      const double ac = a[c];
      for (int e = 0; e < n; ++e) v[e] -= u[e] * ac;
    }
    z.assign(n, 0.0);
    act.assign(n, 0);
    for (int e = 0; e < n; ++e)
      if (v[e] > 0) {
        z[e] = v[e];
        act[e] = 1;
      }
    L.assign(d, 0.0);
    for (int c = 0; c < r; ++c) {
      const double* u = &Um[(size_t)c * n];
      const double* vv = &Vm[(size_t)c * n];
      double s1 = 0, s2 = 0;
      for (int e = 0; e < n; ++e) {
        s1 += u[e] * (y[e] - z[e]);
        s2 += vv[e] * (xt[e] - z[e]);
      }
      L[c] = a[c] + s1;
      L[r + c] = a[r + c] + s2;
    }
  };
  auto infn = [](const Vec& v) {
    double m = 0;
    for (double x : v) m = std::max(m, std::fabs(x));
    return m;
  };
  // semi-smooth Newton from a0 (Alg. 4); returns the residual norm reached
  Vec z;
  int j = 0;
  auto newton = [&](Vec al) -> double {
    Vec L;
    std::vector<char> act;
    residual(al, L, z, act);
    double nr = infn(L);
    std::vector<double> Ua, Va, Ui, UaT, CVaT, CViT;
    int jj;
    for (jj = 0; jj < jmax && nr > tol; ++jj) {
      g_pt.newton++;
      double t_1 = now_s();
      // J = [[U^T Lam U, U^T (I-Lam) CV], [V^T Lam U, -V^T Lam CV]] + I
      std::vector<int> ia, ii;
      for (int e = 0; e < n; ++e) (act[e] ? ia : ii).push_back(e);
      const int na = (int)ia.size(), ni = (int)ii.size();
      // compacted rows (A operands, [r][na|ni]) and transposed columns (B operands, [na|ni][r])
      Ua.assign((size_t)r * na, 0.0);
      Va.assign((size_t)r * na, 0.0);
      Ui.assign((size_t)r * ni, 0.0);
      UaT.assign((size_t)na * r, 0.0);
      CVaT.assign((size_t)na * r, 0.0);
      CViT.assign((size_t)ni * r, 0.0);
#pragma omp parallel for schedule(static) if ((long long)r * n > 1000000)
      for (int c = 0; c < r; ++c) {
        for (int t = 0; t < na; ++t) {
          const double u = Um[(size_t)c * n + ia[t]];
          Ua[(size_t)c * na + t] = u;
          UaT[(size_t)t * r + c] = u;
          Va[(size_t)c * na + t] = Vm[(size_t)c * n + ia[t]];
          CVaT[(size_t)t * r + c] = CV[(size_t)c * n + ia[t]];
        }
        for (int t = 0; t < ni; ++t) {
          Ui[(size_t)c * ni + t] = Um[(size_t)c * n + ii[t]];
          CViT[(size_t)t * r + c] = CV[(size_t)c * n + ii[t]];
        }
      }
      std::vector<double> J((size_t)d * d, 0.0);
      mk_gemm(&J[0], d, Ua.data(), na, UaT.data(), r, r, r, na, false);                   // U^T Lam U
      mk_gemm(&J[r], d, Ui.data(), ni, CViT.data(), r, r, r, ni, false);                  // U^T (I - Lam) CV
      mk_gemm(&J[(size_t)r * d], d, Va.data(), na, UaT.data(), r, r, r, na, false);      // V^T Lam U
      mk_gemm(&J[(size_t)r * d + r], d, Va.data(), na, CVaT.data(), r, r, r, na, true);  // -V^T Lam CV
      for (int i = 0; i < d; ++i) J[(size_t)i * d + i] += 1.0;
      double t_2 = now_s();
      g_pt.jac += t_2 - t_1;
      Vec step = L;
      std::vector<double> Jc = J;
      const bool lu_ok = lu_solve_blocked(Jc, d, step);
      g_pt.lu += now_s() - t_2;
      t_2 = now_s();
      if (!lu_ok) {
        double jn = 0;
        for (double v : J) jn = std::max(jn, std::fabs(v));
        for (int i = 0; i < d; ++i) J[(size_t)i * d + i] += 1e-10 * jn * d;
        step = L;
        if (!lu_solve_blocked(J, d, step)) break;
      }
      double t = 1.0;
      bool ok = false;
      Vec a2(d), L2, z2;
      std::vector<char> act2;
      double n2 = nr;
      for (int h = 0; h < 30; ++h) {
        for (int i = 0; i < d; ++i) a2[i] = al[i] - t * step[i];
        residual(a2, L2, z2, act2);
        n2 = infn(L2);
        if (n2 < nr || n2 <= tol) {
          ok = true;
          break;
        }
        t *= 0.5;
      }
      if (!ok) break;
      double smax = t * infn(step);
      g_pt.resid += now_s() - t_2;
      al = a2;
      L = L2;
      z = z2;
      act = act2;
      nr = n2;
      if (smax < tol) {
        ++jj;
        break;
      }
    }
    j += jj;
    if (nr <= tol) {  // keep the root for the next call on this memory
      q.wc.alpha = al;
      q.wc.alpha_r = r;
    }
    return nr;
  };
  const WoodburyCache& W = q.wc;
  if (W.alpha_r > 0 && W.alpha_r <= r && (int)W.alpha.size() == 2 * W.alpha_r) {
    Vec a0(d, 0.0);
    for (int c = 0; c < W.alpha_r; ++c) {
      a0[c] = W.alpha[c];
      a0[r + c] = W.alpha[W.alpha_r + c];
    }
    if (newton(a0) > tol) newton(Vec(d, 0.0));  // warm start failed: from zero as before
  } else {
    newton(Vec(d, 0.0));
  }
  if (iters) *iters = j;
  return z;
}

// ------------------------------------------------------------------ Alg. 2
double optimal_eta(const Vec& x, const Vec& p, const Vec& g, const Vec& Ap, std::vector<char>& bind) {
  double pAp = dot(p, Ap), pg = dot(p, g);
  double eu = pAp > 0 ? -pg / pAp : std::numeric_limits<double>::infinity();
  double eh = std::numeric_limits<double>::infinity();
  for (size_t i = 0; i < x.size(); ++i)
    if (p[i] < 0) eh = std::min(eh, -x[i] / p[i]);
  bind.assign(x.size(), 0);
  if (eh < eu) {
    for (size_t i = 0; i < x.size(); ++i)
      if (p[i] < 0 && -x[i] / p[i] == eh) bind[i] = 1;
    return eh;
  }
  return eu;
}

// ------------------------------------------------------------------ Alg. 1
// ------------------------------------------------------------------ BB-PGD
// The paper's baseline: x_{k+1} = (x_k - tau_k (A x_k + b))_+ with the
// spectral step tau_bb = |s|^2 / s^T A s of eq. (spectralStepSize), over-relaxation 1
// (Table 1).  tau_0 = 1; a non-positive denominator keeps the previous tau (SPEC
// S:363-365; R31).  One MVP per iteration, on the new iterate.
MonoResult bb_pgd(const MvpFn& mvp, const Vec& b, const Vec& x0, const PqnOpts& o) {
  const size_t n = b.size();
  MonoResult R;
  R.x.resize(n);
  for (size_t i = 0; i < n; ++i) R.x[i] = std::max(x0[i], 0.0);
  Vec Ax;
  mvp(R.x, Ax, nullptr);
  R.mvps = 1;
  R.g.resize(n);
  for (size_t i = 0; i < n; ++i) R.g[i] = Ax[i] + b[i];
  double tau = 1.0, prev = -1.0;
  R.termination = 2;
  for (int k = 0; k < o.k_max; ++k) {
    const double e = kkt_abs(R.x, R.g);
    const double den = prev < 0 ? 0.0 : std::max(e, prev);
    const double erel = prev < 0 ? std::numeric_limits<double>::infinity() : (den > 0 ? std::fabs(e - prev) / den : 0.0);
    prev = e;
    R.kkt = e;
    R.kkt_rel = erel;
    if (e <= o.eps_abs) {
      R.termination = 0;
      break;
    }
    if (o.eps_rel > 0 && erel <= o.eps_rel) {
      R.termination = 1;
      break;
    }
    Vec xn(n), gn(n);
    for (size_t i = 0; i < n; ++i) xn[i] = std::max(R.x[i] - tau * R.g[i], 0.0);
    mvp(xn, Ax, nullptr);
    R.mvps++;
    double ss = 0.0, sAs = 0.0;
    for (size_t i = 0; i < n; ++i) {
      gn[i] = Ax[i] + b[i];
      const double si = xn[i] - R.x[i];
      ss += si * si;
      sAs += si * (gn[i] - R.g[i]);
    }
    if (sAs > 0.0) tau = ss / sAs;
    R.x.swap(xn);
    R.g.swap(gn);
    R.iterations++;
    if (!std::isfinite(tau)) throw std::runtime_error("BB-PGD: non-finite step");
  }
  if (R.termination == 2) R.kkt = kkt_abs(R.x, R.g);
  return R;
}

MonoResult mono_pqn(const MvpFn& mvp, const Vec& b, const Vec& x0, const PqnOpts& o, const Vec* g0,
                    const Vec* aux0, const std::vector<std::pair<Vec, Vec>>* seed) {
  const size_t n = b.size();
  MonoResult R;
  R.x = x0;
  Vec Ax(n), aux(n);
  bool track = false;
  if (!g0) {
    mvp(R.x, Ax, &aux);
    R.mvps++;
    R.g.resize(n);
    for (size_t i = 0; i < n; ++i) R.g[i] = Ax[i] + b[i];
    R.aux = aux;
    track = true;
  } else {
    R.g = *g0;
    if (aux0) {
      R.aux = *aux0;
      track = true;
    }
  }
  Bfgs q;
  if (seed)
    for (auto& sy : *seed) q.update(sy.first, sy.second, nullptr, o.curv);
  double prev = -1;
  bool reset_done = false;
  R.termination = 2;
  int k;
  for (k = 0; k < o.k_max; ++k) {
    double e = kkt_abs(R.x, R.g);
    double rel = prev < 0 ? std::numeric_limits<double>::infinity()
                          : (std::max(e, prev) > 0 ? std::fabs(e - prev) / std::max(e, prev) : 0.0);
    prev = e;
    R.kkt = e;
    R.kkt_rel = rel;
    if (e <= o.eps_abs) {
      R.termination = 0;
      break;
    }
    if (o.eps_rel > 0 && rel <= o.eps_rel) {
      R.termination = 1;
      break;
    }
    Vec hg = q.H(R.g), xt(n);
    for (size_t i = 0; i < n; ++i) xt[i] = R.x[i] - o.tau * hg[i];
    int pit = 0;
    Vec xh = weighted_prox(q, xt, o.prox_tol, o.prox_jmax, &pit);
    Vec p(n);
    for (size_t i = 0; i < n; ++i) p[i] = xh[i] - R.x[i];
    Vec Ap(n), auxp(n);
    mvp(p, Ap, &auxp);
    R.mvps++;
    std::vector<char> bind;
    double eta = optimal_eta(R.x, p, R.g, Ap, bind);
    if (!(eta > 0 && std::isfinite(eta)) || dot(p, R.g) >= 0) {
      if (reset_done) {
        R.termination = 3;
        break;
      }
      q.clear();
      reset_done = true;
      continue;
    }
    reset_done = false;
    for (size_t i = 0; i < n; ++i) {
      R.x[i] += eta * p[i];
      if (bind[i]) R.x[i] = 0.0;
      R.g[i] += eta * Ap[i];
      if (track) R.aux[i] += eta * auxp[i];
    }
    R.iterations++;
    Vec s(n), y(n);
    for (size_t i = 0; i < n; ++i) {
      s[i] = eta * p[i];
      y[i] = eta * Ap[i];
    }
    q.update(s, y, nullptr, o.curv);
    if (o.refresh > 0 && R.iterations % o.refresh == 0) {
      mvp(R.x, Ax, &aux);
      R.mvps++;
      for (size_t i = 0; i < n; ++i) R.g[i] = Ax[i] + b[i];
      if (track) R.aux = aux;
    }
  }
  if (k == o.k_max) R.kkt = kkt_abs(R.x, R.g);
  for (size_t i = 0; i < q.S.size(); ++i) R.pairs.emplace_back(q.S[i], q.Y[i]);
  return R;
}

// ------------------------------------------------------------------ Alg. 3
BiResult bi_pqn(const MvpFn& hi, const MvpFn& lo, const Vec& b, const Vec& x_init, const PqnOpts& o) {
  const size_t n = b.size();
  BiResult R;
  // low-fidelity initialisation: lo MVP returns A^ v, aux = A^ v
  MvpFn lo_aux = [&](const Vec& v, Vec& out, Vec* aux) {
    lo(v, out, nullptr);
    if (aux) *aux = out;
  };
  MonoResult r0 = mono_pqn(lo_aux, b, x_init, o, nullptr, nullptr, nullptr);
  R.lo_mvps += r0.mvps;
  R.init_lo_mvps = r0.mvps;
  Vec x = r0.x, Ahat_x = r0.aux;
  std::vector<std::pair<Vec, Vec>> low = r0.pairs;
  Vec g(n);
  hi(x, g, nullptr);
  R.hi_mvps++;
  for (size_t i = 0; i < n; ++i) g[i] += b[i];
  std::vector<Vec> U, V;
  auto Bhi = [&](const Vec& v, const Vec& Ahat_v) {
    Vec out = Ahat_v;
    for (auto& u : U) {
      double c = dot(u, v);
      for (size_t i = 0; i < n; ++i) out[i] += c * u[i];
    }
    for (auto& w : V) {
      double c = dot(w, v);
      for (size_t i = 0; i < n; ++i) out[i] -= c * w[i];
    }
    return out;
  };
  double prev = -1;
  R.termination = 2;
  int k;
  for (k = 0; k < o.k_max; ++k) {
    double e = kkt_abs(x, g);
    double rel = prev < 0 ? std::numeric_limits<double>::infinity()
                          : (std::max(e, prev) > 0 ? std::fabs(e - prev) / std::max(e, prev) : 0.0);
    prev = e;
    R.kkt = e;
    R.kkt_rel = rel;
    if (e <= o.eps_abs) {
      R.termination = 0;
      break;
    }
    if (o.eps_rel > 0 && rel <= o.eps_rel) {
      R.termination = 1;
      break;
    }
    Vec Bx = Bhi(x, Ahat_x), c(n);
    for (size_t i = 0; i < n; ++i) c[i] = g[i] - Bx[i];
    if (o.verify_secants) {  // max_j |B^(k) s_j - y_j|_inf / max(1, |y_j|_inf), uncounted lo MVPs
      for (auto& sy : low) {
        Vec As(n);
        lo(sy.first, As, nullptr);
        Vec Bs = Bhi(sy.first, As);
        double e = 0, ym = 1.0;
        for (size_t i = 0; i < n; ++i) {
          e = std::max(e, std::fabs(Bs[i] - sy.second[i]));
          ym = std::max(ym, std::fabs(sy.second[i]));
        }
        R.secant_residual = std::max(R.secant_residual, e / ym);
      }
    }
    int sub_lo = 0;
    MvpFn sub = [&](const Vec& v, Vec& out, Vec* aux) {
      Vec Av(n);
      lo(v, Av, nullptr);
      sub_lo++;
      out = Bhi(v, Av);
      if (aux) *aux = Av;
    };
    PqnOpts so = o;
    so.eps_abs = o.sub_eps_factor * o.eps_abs;
    if (o.sub_forcing > 0) so.eps_abs = std::max(so.eps_abs, o.sub_forcing * e);  // inexact subproblems
    so.eps_rel = 0;
    so.k_max = o.sub_k_max;
    MonoResult rs = mono_pqn(sub, c, x, so, &g, &Ahat_x, &low);
    R.lo_mvps += sub_lo;
    R.sub_iterations.push_back(rs.iterations);
    Vec p(n);
    for (size_t i = 0; i < n; ++i) p[i] = rs.x[i] - x[i];
    Vec Ap(n);
    hi(p, Ap, nullptr);
    R.hi_mvps++;
    std::vector<char> bind;
    double eta = optimal_eta(x, p, g, Ap, bind);
    if (!(eta > 0 && std::isfinite(eta))) {
      R.termination = 3;
      break;
    }
    Vec s(n), y(n), Ahat_s(n);
    for (size_t i = 0; i < n; ++i) {
      x[i] += eta * p[i];
      if (bind[i]) x[i] = 0.0;
      g[i] += eta * Ap[i];
      s[i] = eta * p[i];
      y[i] = eta * Ap[i];
      Ahat_s[i] = eta * (rs.aux[i] - Ahat_x[i]);
    }
    R.iterations++;
    Vec Bs = Bhi(s, Ahat_s);
    double ys = dot(y, s), sBs = dot(s, Bs);
    low = rs.pairs;
    if (ys > o.curv * nrm(s) * nrm(y) && sBs > 0) {
      Vec u(n), v(n);
      for (size_t i = 0; i < n; ++i) {
        u[i] = y[i] / std::sqrt(ys);
        v[i] = Bs[i] / std::sqrt(sBs);
      }
      U.push_back(u);
      V.push_back(v);
      // secant re-use: subproblem pairs satisfy B^(k) S = Y; for
      // B^(k+1) = B^(k) + uu^T - vv^T they become Y + (uu^T - vv^T) S (reading R34:
      // the sign the paper's requirement B^(k+1) S = Y fixes, not P:486's display)
      for (auto& sy : low) {
        double cu = dot(u, sy.first), cv = dot(v, sy.first);
        for (size_t i = 0; i < n; ++i) sy.second[i] += cu * u[i] - cv * v[i];
      }
    }
    for (size_t i = 0; i < n; ++i) Ahat_x[i] += Ahat_s[i];
    if (o.refresh > 0 && R.iterations % o.refresh == 0) {
      hi(x, g, nullptr);
      R.hi_mvps++;
      for (size_t i = 0; i < n; ++i) g[i] += b[i];
    }
  }
  if (k == o.k_max) R.kkt = kkt_abs(x, g);
  R.x = x;
  R.g = g;
  R.init_iterations = r0.iterations;
  return R;
}

}  // namespace bpqn
