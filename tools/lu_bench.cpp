// Host micro-benchmark of the prox Newton-system LU (development aid): rank-1 threaded LU vs the
// blocked GEMM-update LU of csrc/pqn.cpp (functions copied verbatim).  g++ -O3 -fopenmp -march=x86-64-v3
#include <vector>
#include <cstdio>
#include <cmath>
#include <random>
#include <chrono>
using Vec = std::vector<double>;
#include <omp.h>
#include <algorithm>
namespace T {
static bool par(long long work) { return work > 200000; }
static void gemm_nt(const double* A, const double* B, double* C, int m, int p, int k, bool acc) {
  const int m2 = m / 2 * 2, p4 = p / 4 * 4;
  auto put = [&](int i, int j, double s) { C[(size_t)i * p + j] = acc ? C[(size_t)i * p + j] + s : s; };
  auto dot = [&](const double* a, const double* b) {
    double s = 0.0;
#pragma omp simd reduction(+ : s)
    for (int e = 0; e < k; ++e) s += a[e] * b[e];
    return s;
  };
#pragma omp parallel for schedule(static) if (par((long long)m * p * k))
  for (int i = 0; i < m2; i += 2) {
    const double* a0 = A + (size_t)i * k;
    const double* a1 = a0 + k;
    for (int j = 0; j < p4; j += 4) {
      const double *b0 = B + (size_t)j * k, *b1 = b0 + k, *b2 = b1 + k, *b3 = b2 + k;
      double s00 = 0, s01 = 0, s02 = 0, s03 = 0, s10 = 0, s11 = 0, s12 = 0, s13 = 0;
#pragma omp simd reduction(+ : s00, s01, s02, s03, s10, s11, s12, s13)
      for (int e = 0; e < k; ++e) {
        const double x0 = a0[e], x1 = a1[e];
        s00 += x0 * b0[e];
        s01 += x0 * b1[e];
        s02 += x0 * b2[e];
        s03 += x0 * b3[e];
        s10 += x1 * b0[e];
        s11 += x1 * b1[e];
        s12 += x1 * b2[e];
        s13 += x1 * b3[e];
      }
      put(i, j, s00);
      put(i, j + 1, s01);
      put(i, j + 2, s02);
      put(i, j + 3, s03);
      put(i + 1, j, s10);
      put(i + 1, j + 1, s11);
      put(i + 1, j + 2, s12);
      put(i + 1, j + 3, s13);
    }
    for (int j = p4; j < p; ++j) {
      put(i, j, dot(a0, B + (size_t)j * k));
      put(i + 1, j, dot(a1, B + (size_t)j * k));
    }
  }
  for (int i = m2; i < m; ++i)
    for (int j = 0; j < p; ++j) put(i, j, dot(A + (size_t)i * k, B + (size_t)j * k));
}
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
    // trailing update A22 -= L21 U12 as one register-blocked GEMM (gemm_nt: C = A B^T with
    // contiguous k = kb rows): L21 and U12^T are copied to contiguous panels first
    const int m = n - k1;
    std::vector<double> Lp((size_t)m * kb), Up((size_t)m * kb), Cp((size_t)m * m);
    for (int i = 0; i < m; ++i)
      for (int k = 0; k < kb; ++k) {
        Lp[(size_t)i * kb + k] = A[(size_t)(k1 + i) * n + k0 + k];
        Up[(size_t)i * kb + k] = A[(size_t)(k0 + k) * n + k1 + i];
      }
    gemm_nt(Lp.data(), Up.data(), Cp.data(), m, m, kb, false);
#pragma omp parallel for schedule(static) if (par((long long)m * m))
    for (int i = 0; i < m; ++i) {
      double* ri = &A[(size_t)(k1 + i) * n + k1];
      const double* ci = &Cp[(size_t)i * m];
#pragma omp simd
      for (int j = 0; j < m; ++j) ri[j] -= ci[j];
    }
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
}
int main(){
  std::mt19937_64 rng(1); std::normal_distribution<double> N(0,1);
  for (int n : {10, 64, 65, 100, 371, 600}) {
    std::vector<double> A(n*n); Vec b(n);
    for (auto& v: A) v = N(rng); for (int i=0;i<n;++i) A[i*n+i]+= 3; for (auto& v: b) v=N(rng);
    auto A1=A, A2=A; Vec b1=b, b2=b;
    auto t0=std::chrono::steady_clock::now(); for(int r=0;r<5;++r){A1=A;b1=b;T::lu_solve_par(A1,n,b1);} auto t1=std::chrono::steady_clock::now();
    for(int r=0;r<5;++r){A2=A;b2=b;T::lu_solve_blocked(A2,n,b2);} auto t2=std::chrono::steady_clock::now();
    double e=0; for(int i=0;i<n;++i) e=std::max(e,std::fabs(b1[i]-b2[i]));
    // residual
    double res=0; for(int i=0;i<n;++i){double s=0; for(int j=0;j<n;++j) s+=A[i*n+j]*b2[j]; res=std::max(res,std::fabs(s-b[i]));}
    printf("n %d diff %.2e resid %.2e  old %.3f ms new %.3f ms\n", n, e, res, std::chrono::duration<double,std::milli>(t1-t0).count()/5, std::chrono::duration<double,std::milli>(t2-t1).count()/5);
  }
}
