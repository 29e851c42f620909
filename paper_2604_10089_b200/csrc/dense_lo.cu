// The low-fidelity LCP matrix densified in HBM (reading R38).
//
// Bi-PQN (Alg. 3) applies the low-fidelity operator A^ = D^T M_lo D hundreds of times
// (c4: ~390 lo MVPs, each a GMRES solve of ~32 iterations at p_lo = 8).  A^ is a fixed Nc x Nc matrix
// for the whole LCP solve, so it can instead be formed once, column by column, with all Nc mobility
// solves running as ONE batched GMRES whose operator application is a dense FP64 GEMM on the tensor
// cores:
//   * the completed double-layer operator A_op = -I/2 + D_full + Pi_R of the handle (K1's coarse
//     stresslet pairs, the refined near rows of K2, the self blocks E_A of K3 -- the same discrete
//     operator, O6/O7) is assembled once as a dense row-major [3N][3N] matrix (c4 at
//     p_lo = 8: 93 312^2 doubles = 69.7 GB of the 180 GB HBM);
//   * right hand sides b_l = -S_full[P^T D e_l] (one single-layer apply per contact);
//   * Nc independent right-preconditioned GMRES(m) processes advance together: per iteration one
//     block-Jacobi GEMM (Minv on every sphere of every column) and one [3N x 3N] x [3N x Nc_active]
//     GEMM (cuBLAS DGEMM, 35 TFLOP/s measured) over the columns not yet converged (gathered
//     contiguously), then one CTA per active column runs its CGS2, Givens rotations and residual;
//     each column stops at its own relative residual tolerance and leaves the GEMMs;
//   * A^ e_l = D^T (-Pi[q_l]) (the rigid read-out and D^T gather of every MVP).
// Every later low-fidelity MVP of the solve is the 540 x 540 product A^ v on the host.  cuBLAS is
// resolved at run time (dlopen; the copy torch loaded when there is one).
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <mutex>
#include <string>
#include <vector>

#include "bpqn_internal.h"

namespace bpqn {

// ---------------------------------------------------------------- cuBLAS (run-time bound)
typedef int (*cublasCreate_t)(void**);
typedef int (*cublasSetStream_t)(void*, cudaStream_t);
typedef int (*cublasDgemm_t)(void*, int, int, int, int, int, const double*, const double*, int, const double*, int,
                             const double*, double*, int);
typedef int (*cublasDtrsm_t)(void*, int, int, int, int, int, int, const double*, const double*, int, double*, int);
typedef int (*cublasDgemmGrouped_t)(void*, const int*, const int*, const int*, const int*, const int*, const double*,
                                    const double* const*, const int*, const double* const*, const int*, const double*,
                                    double* const*, const int*, int, const int*);
struct Cublas {
  cublasCreate_t create = nullptr;
  cublasSetStream_t setStream = nullptr;
  cublasDgemm_t dgemm = nullptr;
  cublasDtrsm_t dtrsm = nullptr;
  cublasDgemmGrouped_t dgemm_grouped = nullptr;  // optional (cuBLAS >= 12.5)
  std::string why;
};
// one cuBLAS handle per calling thread (distinct geometry handles may be used from different threads)
static void* cublas_handle();
static Cublas& cublas() {
  static Cublas c;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libcublas.so.12", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libcublas.so.12", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libcublas.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      c.why = "cuBLAS not found";
      return;
    }
    c.create = reinterpret_cast<cublasCreate_t>(dlsym(h, "cublasCreate_v2"));
    c.setStream = reinterpret_cast<cublasSetStream_t>(dlsym(h, "cublasSetStream_v2"));
    c.dgemm = reinterpret_cast<cublasDgemm_t>(dlsym(h, "cublasDgemm_v2"));
    c.dtrsm = reinterpret_cast<cublasDtrsm_t>(dlsym(h, "cublasDtrsm_v2"));
    c.dgemm_grouped = reinterpret_cast<cublasDgemmGrouped_t>(dlsym(h, "cublasDgemmGroupedBatched"));
    if (!c.create || !c.setStream || !c.dgemm || !c.dtrsm) c.why = "cuBLAS lacks a required symbol";
  });
  if (!c.why.empty()) throw Error{BPQN_ERR_CUDA, c.why};
  return c;
}
static void* cublas_handle() {
  thread_local void* h = nullptr;
  if (!h && cublas().create(&h) != 0) throw Error{BPQN_ERR_CUDA, "cublasCreate failed"};
  return h;
}
constexpr int CUBLAS_OP_N_ = 0, CUBLAS_OP_T_ = 1;

// C[m x n] (col-major, ldc) = op(A) B with A given row-major [m][k] (i.e. col-major A^T, lda = k)
static void gemm_rowA(cudaStream_t st, int m, int n, int k, const double* A_row, const double* B, int ldb, double* C,
                      int ldc, double beta = 0.0) {
  Cublas& cb = cublas();
  void* h = cublas_handle();
  const double one = 1.0;
  if (cb.setStream(h, st) != 0) throw Error{BPQN_ERR_CUDA, "cublasSetStream failed"};
  if (cb.dgemm(h, CUBLAS_OP_T_, CUBLAS_OP_N_, m, n, k, &one, A_row, k, B, ldb, &beta, C, ldc) != 0)
    throw Error{BPQN_ERR_CUDA, "cublasDgemm failed"};
}

// plain column-major DGEMM / DTRSM (cuBLAS conventions)
void blas_dgemm(cudaStream_t st, int ta, int tb, int m, int n, int k, double alpha, const double* A, int lda,
                const double* B, int ldb, double beta, double* C, int ldc) {
  Cublas& cb = cublas();
  void* h = cublas_handle();
  if (cb.setStream(h, st) != 0) throw Error{BPQN_ERR_CUDA, "cublasSetStream failed"};
  if (cb.dgemm(h, ta, tb, m, n, k, &alpha, A, lda, B, ldb, &beta, C, ldc) != 0)
    throw Error{BPQN_ERR_CUDA, "cublasDgemm failed"};
}
constexpr int CB_LEFT = 0, CB_RIGHT = 1, CB_LOWER = 0, CB_NONUNIT = 0;
// G column-major GEMMs C_g = alpha_g A_g B_g (no transposes, beta 0) in one cuBLAS grouped-batched call (one
// problem per group); pointer arrays in device memory.  Returns false if the library lacks the entry point.
bool blas_dgemm_grouped(cudaStream_t st, int G, const int* m, const int* n, const int* k, const double* alpha,
                        const double* const* A_dev, const int* lda, const double* const* B_dev, const int* ldb,
                        double* const* C_dev, const int* ldc) {
  Cublas& cb = cublas();
  if (!cb.dgemm_grouped) return false;
  void* h = cublas_handle();
  if (cb.setStream(h, st) != 0) throw Error{BPQN_ERR_CUDA, "cublasSetStream failed"};
  std::vector<int> tr(G, CUBLAS_OP_N_), one(G, 1);
  std::vector<double> beta(G, 0.0);
  if (cb.dgemm_grouped(h, tr.data(), tr.data(), m, n, k, alpha, A_dev, lda, B_dev, ldb, beta.data(), C_dev, ldc, G,
                       one.data()) != 0)
    throw Error{BPQN_ERR_CUDA, "cublasDgemmGroupedBatched failed"};
  return true;
}

void blas_dtrsm(cudaStream_t st, int side, int trans, int m, int n, const double* L, int ldl, double* B, int ldb) {
  Cublas& cb = cublas();
  void* h = cublas_handle();
  const double one = 1.0;
  if (cb.setStream(h, st) != 0) throw Error{BPQN_ERR_CUDA, "cublasSetStream failed"};
  if (cb.dtrsm(h, side, CB_LOWER, trans, CB_NONUNIT, m, n, &one, L, ldl, B, ldb) != 0)
    throw Error{BPQN_ERR_CUDA, "cublasDtrsm failed"};
}

// ---------------------------------------------------------------- dense operator assembly
// coarse stresslet for every node pair (i, j), i != j:  A[3i+a][3j+b] = -3/(4 pi) w_j (r.n_j) r_a r_b / rho^5
__global__ void k_dense_coarse(int N, const double* __restrict__ src, double* __restrict__ A) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (j >= N) return;
  const double* yi = src + 8 * (size_t)i;
  const double* yj = src + 8 * (size_t)j;
  const double r0 = yi[0] - yj[0], r1 = yi[1] - yj[1], r2 = yi[2] - yj[2];
  const double rr = r0 * r0 + r1 * r1 + r2 * r2;
  double t = 0.0;
  if (i != j) {
    const double rn = r0 * yj[4] + r1 * yj[5] + r2 * yj[6];
    const double ir = 1.0 / sqrt(rr);
    const double ir2 = ir * ir;
    t = -3.0 / (4.0 * 3.14159265358979323846) * yj[3] * rn * ir2 * ir2 * ir;
  }
  const size_t L = 3 * (size_t)N;
  double* row = A + (3 * (size_t)i) * L + 3 * (size_t)j;
  const double r[3] = {r0, r1, r2};
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) row[a * L + b] = t * r[a] * r[b];
}

// near incidences (K2 order pos -> target i, sphere m): the refined rule REPLACES the coarse block:
// A[3i+a][3(m Nq + j)+c] = sum_b T[pos][sym(a,c)][b] analysis[b][j]
__global__ void k_dense_near(int N, int nq, int nb, int nbp, const int* __restrict__ cm_t, const int* __restrict__ cm_m,
                             const double* __restrict__ T, const double* __restrict__ analysis, double* A) {
  const int pos = blockIdx.x;
  const int i = cm_t[pos], m = cm_m[pos];
  extern __shared__ double tr[];  // [6][nb]
  for (int e = threadIdx.x; e < 6 * nb; e += blockDim.x) tr[e] = T[((size_t)pos * 6 + e / nb) * nbp + e % nb];
  __syncthreads();
  const size_t L = 3 * (size_t)N;
  const int sym[3][3] = {{0, 1, 2}, {1, 3, 4}, {2, 4, 5}};
  for (int j = threadIdx.x; j < nq; j += blockDim.x) {
    double s[6] = {0, 0, 0, 0, 0, 0};
    for (int b = 0; b < nb; ++b) {
      const double an = analysis[(size_t)b * nq + j];
#pragma unroll
      for (int q = 0; q < 6; ++q) s[q] = fma(tr[q * nb + b], an, s[q]);
    }
    double* blk = A + (3 * (size_t)i) * L + 3 * ((size_t)m * nq + j);
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) blk[a * L + c] = s[sym[a][c]];
  }
}

// same-sphere blocks: A[3i+a][3(n Nq + j)+c] += E_A[3 il + a][3 j + c]  (E_A = self - naive same-sphere
// stresslet - I/2 + Pi_R, so coarse + E_A = D_self - I/2 + Pi_R)
__global__ void k_dense_self(int N, int nq, const double* __restrict__ EA, double* A) {
  const int i = blockIdx.x;
  const int n = i / nq, il = i - n * nq;
  const size_t L = 3 * (size_t)N;
  const int M = 3 * nq;
  for (int e = threadIdx.x; e < 3 * M; e += blockDim.x) {
    const int a = e / M, col = e - a * M;
    A[(3 * (size_t)i + a) * L + 3 * (size_t)n * nq + col] += EA[(size_t)(3 * il + a) * M + col];
  }
}

// The whole completed double-layer operator A_op of a handle as a dense row-major [3N][3N] matrix in
// a caller-owned device buffer (bpqn_operator_dense; diagnostics and preconditioner studies).
void assemble_dense_operator(Geom& g, double* A, cudaStream_t st) {
  const int N = g.n;
  BPQN_REQUIRE(N <= 65535 && !g.sharded(), "dense operator: N <= 65535 nodes, unsharded handle");
  k_dense_coarse<<<dim3((N + 255) / 256, N), 256, 0, st>>>(N, g.src.p, A);
  BPQN_CHECK_LAUNCH();
  if (g.n_inc > 0) {
    const int nbp = (g.nb + 1) & ~1;
    k_dense_near<<<(unsigned)g.n_inc, 128, 6 * g.nb * sizeof(double), st>>>(N, g.nq, g.nb, nbp, g.cm_t.p, g.cm_m.p,
                                                                             g.T_D.p, g.analysis.p, A);
    BPQN_CHECK_LAUNCH();
  }
  k_dense_self<<<N, 256, 0, st>>>(N, g.nq, g.E_A.p, A);
  BPQN_CHECK_LAUNCH();
}

// ---------------------------------------------------------------- batched GMRES, one CTA per column
struct BgmParams {
  double* V;        // [(m+1)][R][n]
  const double* W;  // [Ra][n] operator output A M^-1 v_k of the active columns (compacted)
  const int* idx;   // [Ra] active column of each CTA
  int n, R, m, k;
  double* H;        // [R][(m+1) m]
  double *cs, *sn, *gv;  // [R][m], [R][m], [R][m+1]
  const double* beta;    // [R] |r0|
  double* resid;         // [R]
};

__device__ __forceinline__ double block_sum(double v, double* sred) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sred[w];
  return s;
}

__global__ void __launch_bounds__(512) k_bgm_step(BgmParams P) {
  __shared__ double sred[16];
  __shared__ double h[2][GM_BATCH_MAX_M + 1];
  const int col = P.idx[blockIdx.x], k = P.k, n = P.n;
  double* w = P.V + ((size_t)(k + 1) * P.R + col) * n;  // z lands in V_{k+1}
  const double* z = P.W + (size_t)blockIdx.x * n;
  for (int e = threadIdx.x; e < n; e += blockDim.x) w[e] = z[e];
  for (int pass = 0; pass < 2; ++pass) {  // CGS2
    for (int i = 0; i <= k; ++i) {
      const double* v = P.V + ((size_t)i * P.R + col) * n;
      double s = 0.0;
      for (int e = threadIdx.x; e < n; e += blockDim.x) s = fma(v[e], w[e], s);
      s = block_sum(s, sred);
      if (threadIdx.x == 0) h[pass][i] = s;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
      double acc = w[e];
      for (int i = 0; i <= k; ++i) acc = fma(-P.V[((size_t)i * P.R + col) * n + e], h[pass][i], acc);
      w[e] = acc;
    }
    __syncthreads();
  }
  double s = 0.0;
  for (int e = threadIdx.x; e < n; e += blockDim.x) s = fma(w[e], w[e], s);
  const double nrm = sqrt(block_sum(s, sred));
  const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
  for (int e = threadIdx.x; e < n; e += blockDim.x) w[e] *= inv;
  if (threadIdx.x != 0) return;
  const int m = P.m;
  double* H = P.H + (size_t)col * (m + 1) * m + (size_t)k * (m + 1);
  double* cs = P.cs + (size_t)col * m;
  double* sn = P.sn + (size_t)col * m;
  double* gv = P.gv + (size_t)col * (m + 1);
  for (int i = 0; i <= k; ++i) H[i] = h[0][i] + h[1][i];
  H[k + 1] = nrm;
  for (int i = 0; i < k; ++i) {
    const double t = cs[i] * H[i] + sn[i] * H[i + 1];
    H[i + 1] = -sn[i] * H[i] + cs[i] * H[i + 1];
    H[i] = t;
  }
  const double den = hypot(H[k], H[k + 1]);
  const double c = den > 0 ? H[k] / den : 1.0, sv = den > 0 ? H[k + 1] / den : 0.0;
  cs[k] = c;
  sn[k] = sv;
  H[k] = den;
  H[k + 1] = 0.0;
  gv[k + 1] = -sv * gv[k];
  gv[k] = c * gv[k];
  P.resid[col] = P.beta[col] > 0.0 ? fabs(gv[k + 1]) / P.beta[col] : 0.0;
}

// V_0 = r / |r| per column; gv = |r| e_1; beta = |r| (relative to the column's |b|: bnorm)
__global__ void k_bgm_start(double* V, const double* r, int n, int m, double* gv, double* beta, double* resid,
                            const double* bnorm) {
  __shared__ double sred[16];
  const int col = blockIdx.x;
  const double* rc = r + (size_t)col * n;
  double s = 0.0;
  for (int e = threadIdx.x; e < n; e += blockDim.x) s = fma(rc[e], rc[e], s);
  const double nr = sqrt(block_sum(s, sred));
  const double inv = nr > 0.0 ? 1.0 / nr : 0.0;
  double* v = V + (size_t)col * n;
  for (int e = threadIdx.x; e < n; e += blockDim.x) v[e] = rc[e] * inv;
  if (threadIdx.x == 0) {
    for (int i = 0; i <= m; ++i) gv[(size_t)col * (m + 1) + i] = 0.0;
    gv[(size_t)col * (m + 1)] = nr;
    const double bn = bnorm ? bnorm[col] : nr;
    beta[col] = bn;  // residuals are relative to |b| (bnorm), as in gmres_solve
    resid[col] = bn > 0.0 ? nr / bn : 0.0;
  }
}

// y = H^-1 gv per column (back substitution, one thread per column); X[:, col] = sum_i y_i V_i
__global__ void k_bgm_backsolve(const double* H, const double* gv, int m, const int* kkv, int R, double* y) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= R) return;
  const int kk = kkv[col];
  const double* Hc = H + (size_t)col * (m + 1) * m;
  double* yc = y + (size_t)col * m;
  for (int i = kk - 1; i >= 0; --i) {
    double acc = gv[(size_t)col * (m + 1) + i];
    for (int j = i + 1; j < kk; ++j) acc -= Hc[(size_t)j * (m + 1) + i] * yc[j];
    yc[i] = Hc[(size_t)i * (m + 1) + i] != 0.0 ? acc / Hc[(size_t)i * (m + 1) + i] : 0.0;
  }
}

__global__ void k_bgm_combine(const double* V, const double* y, int n, int R, int m, const int* kkv, double* X) {
  const int col = blockIdx.y, kk = kkv[col];
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int i = 0; i < kk; ++i) acc = fma(V[((size_t)i * R + col) * n + e], y[(size_t)col * m + i], acc);
    X[(size_t)col * n + e] = acc;
  }
}

// out[:, a] = V[:, idx[a]] (the active columns, contiguous for the GEMMs)
__global__ void k_gather_cols(const double* __restrict__ V, const int* __restrict__ idx, int n, double* __restrict__ out) {
  const double* src = V + (size_t)idx[blockIdx.y] * n;
  double* dst = out + (size_t)blockIdx.y * n;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) dst[e] = src[e];
}

__global__ void k_sub_cols(double* r, const double* b, const double* ax, size_t tot) {
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (size_t)gridDim.x * blockDim.x)
    r[e] = b[e] - ax[e];
}

__global__ void k_col_norms(const double* b, int n, double* out) {
  __shared__ double sred[16];
  const double* bc = b + (size_t)blockIdx.x * n;
  double s = 0.0;
  for (int e = threadIdx.x; e < n; e += blockDim.x) s = fma(bc[e], bc[e], s);
  s = sqrt(block_sum(s, sred));
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}


// ---------------------------------------------------------------- block GMRES (one Krylov space for all columns)
// Lower Cholesky of a column-major n x n SPD block (n <= 64) in shared memory, one CTA; a pivot below
// 1e-28 x the block's largest diagonal entry is clamped there (a rank-deficient block carries no residual).
constexpr int POTRF_NB = 64;
__global__ void __launch_bounds__(256) k_potrf_small(double* A, int n, int lda) {
  __shared__ double a[POTRF_NB][POTRF_NB + 1];
  __shared__ double dmax, dinv;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) a[e / n][e % n] = A[(size_t)(e / n) * lda + e % n];  // a[col][row]
  __syncthreads();
  if (threadIdx.x == 0) {
    double mx = 0.0;
    for (int j = 0; j < n; ++j) mx = fmax(mx, a[j][j]);
    dmax = mx;
  }
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    if (threadIdx.x == 0) {
      const double d = sqrt(fmax(a[j][j], 1e-28 * dmax + 1e-300));
      a[j][j] = d;
      dinv = 1.0 / d;
    }
    __syncthreads();
    for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) a[j][i] *= dinv;
    __syncthreads();
    const int m = n - j - 1;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
      const int i = j + 1 + e % m, l = j + 1 + e / m;
      if (i >= l) a[l][i] -= a[j][i] * a[j][l];
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int l = e / n, i = e % n;
    A[(size_t)l * lda + i] = i >= l ? a[l][i] : 0.0;
  }
}

// C[rows x cols] (ldc) = B (ldb)
__global__ void k_copy_block(double* C, int ldc, const double* B, int ldb, int rows, int cols) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < rows * cols; e += gridDim.x * blockDim.x) {
    const int i = e % rows, j = e / rows;
    C[(size_t)j * ldc + i] = B[(size_t)j * ldb + i];
  }
}

__global__ void k_zero_upper(double* A, int n, int lda) {
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < (size_t)n * n; e += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % n), l = (int)(e / n);
    if (i < l) A[(size_t)l * lda + i] = 0.0;
  }
}

static int grid_for(size_t work) { return (int)std::max<size_t>(1, std::min<size_t>((work + 255) / 256, 4096)); }

// Blocked right-looking Cholesky A = L L^T (column-major, lower, the strict upper triangle zeroed): panels of 64 in shared memory, the
// panel below by DTRSM and the trailing update by DGEMM (cuBLAS).
void dev_potrf(cudaStream_t st, double* A, int n, int lda) {
  for (int j = 0; j < n; j += POTRF_NB) {
    const int jb = std::min(POTRF_NB, n - j);
    double* Ajj = A + (size_t)j * lda + j;
    k_potrf_small<<<1, 256, 0, st>>>(Ajj, jb, lda);
    BPQN_CHECK_LAUNCH();
    const int r = n - j - jb;
    if (r > 0) {
      double* P = Ajj + jb;  // rows j+jb.., columns j..j+jb
      blas_dtrsm(st, CB_RIGHT, CUBLAS_OP_T_, r, jb, Ajj, lda, P, lda);
      blas_dgemm(st, CUBLAS_OP_N_, CUBLAS_OP_T_, r, r, jb, -1.0, P, lda, P, lda, 1.0, Ajj + (size_t)jb * lda + jb, lda);
    }
  }
  k_zero_upper<<<grid_for((size_t)n * n), 256, 0, st>>>(A, n, lda);
  BPQN_CHECK_LAUNCH();
}

// C[rows x cols] (ldc) += B[rows x cols] (ldb)
__global__ void k_add_block(double* C, int ldc, const double* B, int ldb, int rows, int cols) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < rows * cols; e += gridDim.x * blockDim.x) {
    const int i = e % rows, j = e / rows;
    C[(size_t)j * ldc + i] += B[(size_t)j * ldb + i];
  }
}

// C[rows x cols] (ldc) = B^T, B [cols x rows] (ldb)
__global__ void k_transpose_block(double* C, int ldc, const double* B, int ldb, int rows, int cols) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < rows * cols; e += gridDim.x * blockDim.x) {
    const int i = e % rows, j = e / rows;
    C[(size_t)j * ldc + i] = B[(size_t)i * ldb + j];
  }
}

// column norms of a column-major [n x cols] block (ld) relative to bnorm: out[c] = |X[:, c]| / bnorm[c]
__global__ void k_col_rel_norms(const double* X, int n, int ld, const double* bnorm, double* out) {
  __shared__ double sred[32];
  const double* xc = X + (size_t)blockIdx.x * ld;
  double s = 0.0;
  for (int e = threadIdx.x; e < n; e += blockDim.x) s = fma(xc[e], xc[e], s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sred[w];
    const double bn = bnorm[blockIdx.x];
    out[blockIdx.x] = bn > 0.0 ? sqrt(t) / bn : 0.0;
  }
}

// ---------------------------------------------------------------- driver
// Right-preconditioned block GMRES for all R columns at once (one Krylov space of dimension R per block
// iteration; the columns share the operator's slow modes, so far fewer operator applications than R
// independent GMRES processes: c4 lo 23 block iterations against 42, tools/block_gmres_study.py):
//   * block Arnoldi with block CGS2 (DGEMM) and Cholesky-QR2 of each new block (blocked Cholesky in
//     shared memory + DTRSM/DGEMM), so V_{k+1} H_{k+1,k} = W with H_{k+1,k} upper triangular;
//   * the least-squares problem min |E1 S0 - Hbar Y| of every column by the normal equations of Hbar,
//     whose Cholesky factor grows by one block row per iteration (DTRSM + a 64-panel Cholesky), with one
//     step of refinement from the explicit residual (corrected semi-normal equations);
//   * every column's explicit LS residual relative to its |b| decides convergence; restarted every kmax
//     block iterations from the true residual b - A x.
// X (x0 = 0 on entry) receives M^-1 V Y, the density of each column.
static int block_gmres(Geom& g, const double* A, const double* B, const double* BN, double* X, int R, size_t n,
                       int kmax, double tol, int max_blocks, cudaStream_t st, long long& col_iters) {
  const int s = R, M3 = 3 * g.nq;
  const int ldH = (kmax + 1) * s, ldL = kmax * s;
  DBuf<double> V, H, L, F, Y, Y2, Res, Tb, Gs, G2, Z, Wt, S0, RES;
  V.alloc((size_t)(kmax + 1) * s * n);
  H.alloc((size_t)ldH * ldL);
  L.alloc((size_t)ldL * ldL);
  F.alloc((size_t)ldL * s);
  Y.alloc((size_t)ldL * s);
  Y2.alloc((size_t)ldL * s);
  Res.alloc((size_t)ldH * s);
  Tb.alloc((size_t)ldH * s);
  Gs.alloc((size_t)s * s);
  G2.alloc((size_t)s * s);
  Z.alloc((size_t)s * n);
  Wt.alloc((size_t)s * n);
  S0.alloc((size_t)s * s);
  RES.alloc(s);
  const int T_ = CUBLAS_OP_T_, N_ = CUBLAS_OP_N_;
  // W = Q R with Q overwriting W, R = (L1 L2)^T upper (ld ldr)
  auto cholqr2 = [&](double* W, double* Rout, int ldr) {
    blas_dgemm(st, T_, N_, s, s, (int)n, 1.0, W, (int)n, W, (int)n, 0.0, Gs.p, s);
    dev_potrf(st, Gs.p, s, s);
    blas_dtrsm(st, CB_RIGHT, T_, (int)n, s, Gs.p, s, W, (int)n);
    blas_dgemm(st, T_, N_, s, s, (int)n, 1.0, W, (int)n, W, (int)n, 0.0, G2.p, s);
    dev_potrf(st, G2.p, s, s);
    blas_dtrsm(st, CB_RIGHT, T_, (int)n, s, G2.p, s, W, (int)n);
    blas_dgemm(st, T_, T_, s, s, s, 1.0, G2.p, s, Gs.p, s, 0.0, Rout, ldr);  // L2^T L1^T
  };
  // Res = E1 S0 - Hbar[0:kk+s, 0:kk] Y  (ld ldH)
  auto residual = [&](int kk, const double* Yp) {
    BPQN_CUDA(cudaMemsetAsync(Res.p, 0, 8 * (size_t)ldH * s, st));
    k_copy_block<<<grid_for((size_t)s * s), 256, 0, st>>>(Res.p, ldH, S0.p, s, s, s);
    BPQN_CHECK_LAUNCH();
    blas_dgemm(st, N_, N_, kk + s, s, kk, -1.0, H.p, ldH, Yp, ldL, 1.0, Res.p, ldH);
  };
  auto cholsolve = [&](int kk, double* Yp) {  // Yp <- (L L^T)^-1 Yp on the leading kk rows
    blas_dtrsm(st, CB_LEFT, N_, kk, s, L.p, ldL, Yp, ldL);
    blas_dtrsm(st, CB_LEFT, T_, kk, s, L.p, ldL, Yp, ldL);
  };
  std::vector<double> res(s);
  int total = 0;
  bool first = true;
  for (;;) {
    double* V0 = V.p;
    if (first) {
      BPQN_CUDA(cudaMemcpyAsync(V0, B, 8 * (size_t)s * n, cudaMemcpyDeviceToDevice, st));
    } else {  // restart from the true residual b - A_op x
      gemm_rowA(st, (int)n, s, (int)n, A, X, (int)n, Wt.p, (int)n);
      k_sub_cols<<<grid_for((size_t)s * n), 256, 0, st>>>(V0, B, Wt.p, (size_t)s * n);
      BPQN_CHECK_LAUNCH();
    }
    first = false;
    cholqr2(V0, S0.p, s);
    BPQN_CUDA(cudaMemsetAsync(H.p, 0, 8 * (size_t)ldH * ldL, st));
    bool done = false;
    for (int k = 0; k < kmax; ++k) {
      double* Vk = V.p + (size_t)k * s * n;
      double* Vn = Vk + (size_t)s * n;
      double* Hk = H.p + (size_t)k * s * ldH;
      const int kk = (k + 1) * s;
      // W = A_op M^-1 V_k (block-Jacobi GEMM over all spheres of all columns, then the dense operator)
      gemm_rowA(st, M3, g.np * s, M3, g.Minv.p, Vk, M3, Z.p, M3);
      gemm_rowA(st, (int)n, s, (int)n, A, Z.p, (int)n, Vn, (int)n);
      // block CGS2 against V_0..V_k
      blas_dgemm(st, T_, N_, kk, s, (int)n, 1.0, V.p, (int)n, Vn, (int)n, 0.0, Hk, ldH);
      blas_dgemm(st, N_, N_, (int)n, s, kk, -1.0, V.p, (int)n, Hk, ldH, 1.0, Vn, (int)n);
      blas_dgemm(st, T_, N_, kk, s, (int)n, 1.0, V.p, (int)n, Vn, (int)n, 0.0, Tb.p, kk);
      blas_dgemm(st, N_, N_, (int)n, s, kk, -1.0, V.p, (int)n, Tb.p, kk, 1.0, Vn, (int)n);
      k_add_block<<<grid_for((size_t)kk * s), 256, 0, st>>>(Hk, ldH, Tb.p, kk, kk, s);
      BPQN_CHECK_LAUNCH();
      cholqr2(Vn, Hk + kk, ldH);  // H_{k+1,k}
      // normal equations: new block column of Hbar^T Hbar, then block row k of its Cholesky factor
      blas_dgemm(st, T_, N_, kk, s, kk + s, 1.0, H.p, ldH, Hk, ldH, 0.0, Tb.p, kk);
      double* Lkk = L.p + (size_t)k * s * ldL + (size_t)k * s;
      if (k > 0) {
        blas_dtrsm(st, CB_LEFT, N_, k * s, s, L.p, ldL, Tb.p, kk);                           // X = L^-1 G[0:ks, k]
        blas_dgemm(st, T_, N_, s, s, k * s, -1.0, Tb.p, kk, Tb.p, kk, 1.0, Tb.p + (size_t)k * s, kk);  // G_kk - X^T X
        k_transpose_block<<<grid_for((size_t)s * k * s), 256, 0, st>>>(L.p + (size_t)k * s, ldL, Tb.p, kk, s, k * s);
        BPQN_CHECK_LAUNCH();
      }
      k_copy_block<<<grid_for((size_t)s * s), 256, 0, st>>>(Lkk, ldL, Tb.p + (size_t)k * s, kk, s, s);
      BPQN_CHECK_LAUNCH();
      dev_potrf(st, Lkk, s, ldL);
      // F block k = Hbar[0:s, block k]^T S0 (E1 S0 is zero below the first block row)
      blas_dgemm(st, T_, N_, s, s, s, 1.0, Hk, ldH, S0.p, s, 0.0, F.p + (size_t)k * s, ldL);
      // Y = (L L^T)^-1 F, one refinement step from the explicit residual
      k_copy_block<<<grid_for((size_t)kk * s), 256, 0, st>>>(Y.p, ldL, F.p, ldL, kk, s);
      BPQN_CHECK_LAUNCH();
      cholsolve(kk, Y.p);
      residual(kk, Y.p);
      blas_dgemm(st, T_, N_, kk, s, kk + s, 1.0, H.p, ldH, Res.p, ldH, 0.0, Y2.p, ldL);
      cholsolve(kk, Y2.p);
      k_add_block<<<grid_for((size_t)kk * s), 256, 0, st>>>(Y.p, ldL, Y2.p, ldL, kk, s);
      BPQN_CHECK_LAUNCH();
      residual(kk, Y.p);
      k_col_rel_norms<<<s, 256, 0, st>>>(Res.p, kk + s, ldH, BN, RES.p);
      BPQN_CHECK_LAUNCH();
      BPQN_CUDA(cudaMemcpyAsync(res.data(), RES.p, 8 * (size_t)s, cudaMemcpyDeviceToHost, st));
      BPQN_CUDA(cudaStreamSynchronize(st));
      ++total;
      col_iters += s;
      double worst = 0.0;
      for (double v : res) {
        if (!std::isfinite(v)) throw Error{BPQN_ERR_NAN, "NaN in the block low-fidelity GMRES"};
        worst = std::max(worst, v);
      }
      done = worst <= tol;
      if (done || k + 1 == kmax || total >= max_blocks) {  // x += M^-1 V_{0..k} Y
        blas_dgemm(st, N_, N_, (int)n, s, kk, 1.0, V.p, (int)n, Y.p, ldL, 0.0, Wt.p, (int)n);
        gemm_rowA(st, M3, g.np * s, M3, g.Minv.p, Wt.p, M3, X, M3, 1.0);
        break;
      }
    }
    if (done) return total;
    if (total >= max_blocks) throw Error{BPQN_ERR_NOCONV, "block low-fidelity GMRES did not converge"};
  }
}

size_t dense_lo_bytes(const Geom& g, int m) {
  const size_t n = 3 * (size_t)g.n, R = (size_t)std::max(g.nc, 1);
  return 8 * (n * n + (size_t)(m + 1) * R * n + 4 * R * n);
}
// block GMRES with kmax block iterations per cycle: operator, V, Hbar, L, and the [n x R] buffers
static size_t dense_lo_block_bytes(const Geom& g, int kmax) {
  const size_t n = 3 * (size_t)g.n, R = (size_t)std::max(g.nc, 1), K = (size_t)kmax;
  return 8 * (n * n + (K + 1) * R * n + (K + 1) * R * K * R + K * R * K * R + 6 * R * n + 6 * K * R * R);
}

int densify_lcp(Geom& g, const bpqn_gmres_opts& o, std::vector<double>& Ahat, DenseLoStats& stt, cudaStream_t st) {
  const auto t0 = std::chrono::steady_clock::now();
  const int N = g.n, R = g.nc, nq = g.nq;
  const size_t n = 3 * (size_t)N;
  BPQN_REQUIRE(R > 0, "no contacts installed");
  BPQN_REQUIRE(N <= 65535 && !g.sharded(), "dense low fidelity: N <= 65535 nodes, unsharded handle");
  BPQN_REQUIRE(g.Minv.p && g.E_A.p, "geometry has no self operators");
  size_t fr = 0, tot = 0;
  BPQN_CUDA(cudaMemGetInfo(&fr, &tot));
  // block GMRES or the batched per-column GMRES.  Block CGS2 costs ~8 k s^2 n flops per block iteration
  // against 2 n^2 s for the operator, so the block form pays when n >> s (measured: c4 lo n = 173 s,
  // block 9.8 s vs batched 12.6 s; c4 centres at p = 4, n = 48 s, block 1.43 s vs batched 1.17 s):
  // block when n >= 100 s; BPQN_LO_BATCHED=1 / BPQN_LO_BLOCK=1 force either.
  const char* eb = getenv("BPQN_LO_BATCHED");
  const char* ek = getenv("BPQN_LO_BLOCK");
  const bool blockmode = (ek && ek[0] == '1') || (!(eb && eb[0] == '1') && n >= (size_t)100 * R);
  int m = std::max(4, std::min(o.restart, GM_BATCH_MAX_M));
  int kmax = std::max(2, std::min(40, (int)(n / std::max(R, 1)) - 1));
  if (const char* ek = getenv("BPQN_LO_BLOCK_KMAX")) kmax = std::max(1, std::min(kmax, atoi(ek)));  // tests: restarts
  if (blockmode) {
    while (kmax > 4 && dense_lo_block_bytes(g, kmax) + ((size_t)1 << 30) > fr) kmax -= 4;
    if (dense_lo_block_bytes(g, kmax) + ((size_t)1 << 30) > fr)
      throw Error{BPQN_ERR_OOM, "dense low-fidelity operator does not fit in device memory"};
  } else {
    while (m > 8 && dense_lo_bytes(g, m) + ((size_t)1 << 30) > fr) m /= 2;
    if (dense_lo_bytes(g, m) + ((size_t)1 << 30) > fr)
      throw Error{BPQN_ERR_OOM, "dense low-fidelity operator does not fit in device memory"};
  }
  cublas_handle();  // fail early if cuBLAS is missing
  DBuf<double> A, V, B, Wb, X, Z, G, sm;
  DBuf<int> didx, dkk;
  A.alloc(n * n);
  B.alloc((size_t)R * n);
  X.alloc((size_t)R * n);
  DBuf<double> bn_blk;
  bn_blk.alloc(R);
  double* BN = bn_blk.p;
  // 1. assemble A_op (coarse -> near rows replace -> self blocks add)
  assemble_dense_operator(g, A.p, st);
  // 2. right-hand sides b_l = -S[P^T D e_l]
  BPQN_REQUIRE(g.E_S.p, "geometry built without single-layer data");
  DBuf<double> eye;
  {
    std::vector<double> I((size_t)R * R, 0.0);
    for (int l = 0; l < R; ++l) I[(size_t)l * R + l] = 1.0;
    eye.alloc(I.size());
    BPQN_CUDA(cudaMemcpyAsync(eye.p, I.data(), 8 * I.size(), cudaMemcpyHostToDevice, st));
    BPQN_CUDA(cudaStreamSynchronize(st));
  }
  for (int l = 0; l < R; ++l) {
    launch_d_scatter(g, eye.p + (size_t)l * R, g.ft.p, st);
    launch_pt(g, g.ft.p, g.tmp.p, st);
    apply_operator(g, g.tmp.p, nullptr, g.E_S.p, nullptr, B.p + (size_t)l * n, st);
  }
  launch_axpby(B.p, 0.0, B.p, -1.0, (size_t)R * n, st);
  k_col_norms<<<R, 512, 0, st>>>(B.p, (int)n, BN);
  BPQN_CHECK_LAUNCH();
  const auto t1 = std::chrono::steady_clock::now();
  BPQN_CUDA(cudaMemsetAsync(X.p, 0, 8 * (size_t)R * n, st));
  int iters = 0;
  long long col_iters = 0;
  if (blockmode) {
    iters = block_gmres(g, A.p, B.p, BN, X.p, R, n, kmax, o.tol, std::max(1, o.max_iters), st, col_iters);
    m = kmax;
  } else {
  G.alloc((size_t)R * n);
  didx.alloc(R);
  dkk.alloc(R);
  V.alloc((size_t)(m + 1) * R * n);
  Wb.alloc((size_t)R * n);
  Z.alloc((size_t)R * n);
  const size_t hs = (size_t)R * (m + 1) * m, cs = (size_t)R * m, gs = (size_t)R * (m + 1);
  sm.alloc(hs + 3 * cs + gs + 3 * (size_t)R);
  double *H = sm.p, *CS = H + hs, *SN = CS + cs, *Y = SN + cs, *GV = Y + cs, *BETA = GV + gs, *RES = BETA + R;
  // 3. batched right-preconditioned GMRES(m), x0 = 0
  const int M3 = 3 * nq;
  auto apply_op = [&](const double* in, int ncol, double* out) {  // out = A_op Minv in (ncol columns)
    gemm_rowA(st, M3, g.np * ncol, M3, g.Minv.p, in, M3, Z.p, M3);
    gemm_rowA(st, (int)n, ncol, (int)n, A.p, Z.p, (int)n, out, (int)n);
  };
  std::vector<double> res(R);
  std::vector<int> active, kkc(R);
  bool first = true, done = false;
  while (!done) {
    const double* r0 = B.p;
    if (!first) {  // restart: r = b - A x  (x holds the solution so far, already M^-1 applied)
      gemm_rowA(st, (int)n, R, (int)n, A.p, X.p, (int)n, Wb.p, (int)n);
      k_sub_cols<<<std::min<int>((int)(((size_t)R * n + 255) / 256), g.sms * 16), 256, 0, st>>>(Wb.p, B.p, Wb.p,
                                                                                            (size_t)R * n);
      r0 = Wb.p;
    }
    first = false;
    k_bgm_start<<<R, 512, 0, st>>>(V.p, r0, (int)n, m, GV, BETA, RES, BN);
    BPQN_CHECK_LAUNCH();
    // columns already at tolerance (a restart) take no step; the others are compacted for the GEMMs
    BPQN_CUDA(cudaMemcpyAsync(res.data(), RES, 8 * (size_t)R, cudaMemcpyDeviceToHost, st));
    BPQN_CUDA(cudaStreamSynchronize(st));
    active.clear();
    for (int c = 0; c < R; ++c) {
      kkc[c] = 0;
      if (!(res[c] <= o.tol)) active.push_back(c);
    }
    for (int k = 0; k < m && !active.empty(); ++k) {
      const int Ra = (int)active.size();
      BPQN_CUDA(cudaMemcpyAsync(didx.p, active.data(), 4 * (size_t)Ra, cudaMemcpyHostToDevice, st));
      k_gather_cols<<<dim3(std::max(1, std::min<int>((int)((n + 255) / 256), 32)), Ra), 256, 0, st>>>(
          V.p + (size_t)k * R * n, didx.p, (int)n, G.p);
      apply_op(G.p, Ra, Wb.p);
      BgmParams P{V.p, Wb.p, didx.p, (int)n, R, m, k, H, CS, SN, GV, BETA, RES};
      k_bgm_step<<<Ra, 512, 0, st>>>(P);
      BPQN_CHECK_LAUNCH();
      ++iters;
      col_iters += Ra;
      BPQN_CUDA(cudaMemcpyAsync(res.data(), RES, 8 * (size_t)R, cudaMemcpyDeviceToHost, st));
      BPQN_CUDA(cudaStreamSynchronize(st));
      std::vector<int> still;
      for (int c : active) {
        if (!std::isfinite(res[c])) throw Error{BPQN_ERR_NAN, "NaN in the batched low-fidelity GMRES"};
        kkc[c] = k + 1;
        if (res[c] > o.tol) still.push_back(c);
      }
      active.swap(still);
      if (active.empty()) done = true;
      else if (iters >= o.max_iters) throw Error{BPQN_ERR_NOCONV, "batched low-fidelity GMRES did not converge"};
    }
    if (active.empty()) done = true;
    // x += M^-1 V y, each column with its own step count
    BPQN_CUDA(cudaMemcpyAsync(dkk.p, kkc.data(), 4 * (size_t)R, cudaMemcpyHostToDevice, st));
    k_bgm_backsolve<<<(R + 127) / 128, 128, 0, st>>>(H, GV, m, dkk.p, R, Y);
    k_bgm_combine<<<dim3(std::max(1, std::min<int>((int)((n + 255) / 256), 64)), R), 256, 0, st>>>(V.p, Y, (int)n, R,
                                                                                                   m, dkk.p, Wb.p);
    BPQN_CHECK_LAUNCH();
    gemm_rowA(st, M3, g.np * R, M3, g.Minv.p, Wb.p, M3, X.p, M3, 1.0);
  }
  }  // batched
  // 4. A^ e_l = D^T (-Pi[q_l])
  DBuf<double> Ad;
  Ad.alloc((size_t)R * R);
  for (int l = 0; l < R; ++l) {
    launch_rigid_readout(g, X.p + (size_t)l * n, g.uo.p, st);
    launch_dt_gather(g, g.uo.p, Ad.p + (size_t)l * R, 1.0, nullptr, st);
  }
  std::vector<double> colmajor((size_t)R * R);
  BPQN_CUDA(cudaMemcpyAsync(colmajor.data(), Ad.p, 8 * (size_t)R * R, cudaMemcpyDeviceToHost, st));
  BPQN_CUDA(cudaStreamSynchronize(st));
  Ahat.assign((size_t)R * R, 0.0);  // row-major A^[i][l] = column l, entry i
  for (int l = 0; l < R; ++l)
    for (int i = 0; i < R; ++i) Ahat[(size_t)i * R + l] = colmajor[(size_t)l * R + i];
  const auto t2 = std::chrono::steady_clock::now();
  stt.columns = R;
  stt.iters = iters;
  stt.col_iters = col_iters;
  stt.restart = m;
  stt.ms_rhs = std::chrono::duration<double, std::milli>(t1 - t0).count();
  stt.ms_total = std::chrono::duration<double, std::milli>(t2 - t0).count();
  stt.bytes = blockmode ? dense_lo_block_bytes(g, kmax) : dense_lo_bytes(g, m);
  return BPQN_OK;
}

}  // namespace bpqn
