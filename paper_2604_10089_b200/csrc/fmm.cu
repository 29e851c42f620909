// Far-field acceleration of K1 for N >> 3e5 ("an FMM for N >> 3x10^5"; the paper's far field
// is an OpenMP Stokes FMM): a kernel-independent FMM on a uniform octree.
//
// It approximates exactly what K1 computes -- the coarse-rule Stokeslet / stresslet sum over every node
// pair i != j,  u_i = sum_j cS w_j (f_j / rho + (r.f_j) r / rho^3) + cD w_j (r.n_j)(r.q_j) r / rho^5 -- so
// K2 (near rows) and K3 (self blocks) apply unchanged on top of it.  Per box of half-width r the far
// field is carried by Stokeslet equivalent densities on cube surfaces (order p_e points per edge):
// upward equivalent at 1.05 r / check at 2.95 r, downward check at 1.05 r / equivalent at 2.95 r; each
// check-to-equivalent map is the Tikhonov-regularised pseudo-inverse of the Stokeslet matrix between the
// two surfaces (normal equations, blocked Cholesky on the device).  Every translation is a dense
// [3 n_s x 3 n_s] matrix computed once for a unit box and scaled per level by the Stokeslet's
// homogeneity (G(s x) = G(x) / s): M2M and L2L per child octant, M2L per interaction offset (316), all
// applied as cuBLAS DGEMMs (FP64 tensor cores) over the occupied boxes of a level.  Leaves: P2M and the
// near field (27 neighbour leaves, i != j) by direct sums, L2P by the leaf's downward equivalent density.
// Every accumulation has a fixed order (octants, then offsets, per target box): bit-reproducible.
// Accuracy is set by p_e (measured against the direct sum, tests and profiles/r02_fmm.md).
#include <algorithm>
#include <cmath>
#include <vector>

#include "bpqn_internal.h"

namespace bpqn {

constexpr double FMM_IN = 1.05, FMM_OUT = 2.95;  // surface radii (box half-widths)
constexpr int FMM_NOFF = 316;
constexpr int FMM_OP_N = 0, FMM_OP_T = 1;

struct FmmLevel {
  int nocc = 0;
  double r = 0.0;
  std::vector<int> dense;   // compact -> dense box index
  DBuf<double> ctr;         // [nocc][3] box centres
  DBuf<double> ueq, uck, deq, dck;  // [nocc] columns of 3 n_s
  // this level as parent: per child octant the (parent, child) compact pairs
  int n_oct[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  DBuf<int> oct_par[8], oct_ch[8];
  // the same pairs octant-major in one list (column j of the gathered buffers), the parents' CSR over the
  // columns (octant order), and the 8 octant GEMMs of M2M / L2L as grouped-batched cuBLAS calls
  int n_child = 0;
  int oct_start[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  DBuf<int> par_all, ch_all, par_ptr, par_pos;
  std::vector<int> mm_m, mm_n, mm_k, mm_lda, mm_ldb, mm_ldc, ll_k, ll_ldb;
  std::vector<double> mm_alpha;
  DBuf<const double*> mm_A, mm_B, ll_A, ll_B;
  DBuf<double*> mm_C;
  // M2L into this level: pairs in offset-major order (source compact ids), offset ranges, and per target
  // the pair positions in offset order (CSR)
  int n_pairs = 0;
  std::vector<int> off_start;  // [FMM_NOFF + 1]
  DBuf<int> m2l_src, tgt_ptr, tgt_pos;
  // the level's M2L GEMMs as one grouped-batched cuBLAS call: per non-empty offset the sizes and the
  // device pointers of (M2L_o, its gathered sources, its outputs)
  std::vector<int> g_m, g_n, g_k, g_lda, g_ldb, g_ldc;
  std::vector<double> g_alpha;
  DBuf<const double*> g_A, g_B;
  DBuf<double*> g_C;
  void reset() {
    nocc = 0;
    r = 0.0;
    dense.clear();
    off_start.clear();
    n_pairs = 0;
    for (int o = 0; o < 8; ++o) n_oct[o] = 0;
    n_child = 0;
  }
};

struct Fmm {
  int pe = 0, ns = 0, L = 0;
  double lo[3] = {0, 0, 0}, R0 = 1.0;
  FmmLevel lev[8];               // levels 0..L (L <= 7)
  DBuf<double> surf;             // [ns][3] unit cube surface points
  DBuf<double> UC2E, DC2E;       // [3ns][3ns] (unit box)
  DBuf<double> M2M, L2L;         // [8][3ns][3ns]
  DBuf<double> M2L;              // [316][3ns][3ns + 1]
  // compressed M2L (low orders): M2L_o ~ WU M2L_o[I, J] WV^T with one row skeleton I and one column skeleton J
  // for all 316 offsets (interpolative decompositions by pivoted Cholesky of the two Gram matrices)
  bool m2l_comp = false;
  int rU = 0, rV = 0;
  DBuf<double> WU, WV;           // [3ns][rU], [3ns + 1][rV] (column-major)
  DBuf<double> M2Lc;             // [316][rU][rV]
  std::vector<int> offs;         // [316][3]
  DBuf<int> perm;                // [N] sorted position -> node
  DBuf<int> leaf_start;          // [nleaf + 1]
  DBuf<int> leaf_nbr;            // [nleaf][27]
  DBuf<double> rec;              // [N][12] sorted records {y, n, f~, q~}
  // small leaves: the near field + L2P as equal-cost items (leaf, 64-target chunk, source segment), see
  // k_fmm_leaf_seg; part[s][k][3] = segment s's sum for sorted target k, tparts[k] = its number of segments
  DBuf<int> leaf_items;          // [n_items][4] = {leaf, chunk, segment, segment length}
  DBuf<int> tparts;              // [N]
  DBuf<double> part;             // [kmax][N][3]
  int n_items = 0, n_near = 0, kmax = 0;  // items [0, n_near): near-field segments, [n_near, n_items): L2P
  // the tree pass (P2M ... L2L, small GEMMs and gathers that leave the FP64 pipe half idle) runs on a
  // high-priority side stream while the near-field items run on the caller's stream
  cudaStream_t tree_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  ~Fmm() {
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (tree_stream) cudaStreamDestroy(tree_stream);
  }
  DBuf<double> bufB, bufC, tmpA, tmpB;
  size_t buf_cols = 0;
  bool ops_ready = false;
};

void fmm_free(Fmm* f) { delete f; }

template <class T>
static void fmm_upload(DBuf<T>& d, const std::vector<T>& h, cudaStream_t st) {
  d.alloc(h.size());
  if (!h.empty()) BPQN_CUDA(cudaMemcpyAsync(d.p, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice, st));
}

// ------------------------------------------------------------------ kernels
// K[3i + a][3j + b] (column-major, ld) = G_ab(x_i - y_j), G = I / rho + r r^T / rho^3; points scaled / shifted:
// x_i = sx * tx[i] + ox, y_j = sy * ty[j] + oy
__global__ void k_fmm_gmat(const double* __restrict__ tx, int m, double sx, double3 ox, const double* __restrict__ ty,
                           int n, double sy, double3 oy, double* __restrict__ K, int ld) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  if (i >= m) return;
  const double r0 = (sx * tx[3 * i] + ox.x) - (sy * ty[3 * j] + oy.x);
  const double r1 = (sx * tx[3 * i + 1] + ox.y) - (sy * ty[3 * j + 1] + oy.y);
  const double r2 = (sx * tx[3 * i + 2] + ox.z) - (sy * ty[3 * j + 2] + oy.z);
  const double ir = 1.0 / sqrt(r0 * r0 + r1 * r1 + r2 * r2), ir3 = ir * ir * ir;
  const double r[3] = {r0, r1, r2};
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) K[(size_t)(3 * j + b) * ld + 3 * i + a] = (a == b ? ir : 0.0) + r[a] * r[b] * ir3;
}

// one extra column: the velocity of a point source at y (potential flow, u = fac (x - y) / |x - y|^3) -- the
// net flux of stresslet sources, which no Stokeslet (divergence-free) equivalent density carries
__global__ void k_fmm_srccol(const double* __restrict__ tx, int m, double sx, double3 ox, double3 y, double fac,
                             double* __restrict__ col) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const double r0 = sx * tx[3 * i] + ox.x - y.x, r1 = sx * tx[3 * i + 1] + ox.y - y.y, r2 = sx * tx[3 * i + 2] + ox.z - y.z;
  const double ir = 1.0 / sqrt(r0 * r0 + r1 * r1 + r2 * r2), ir3 = fac * ir * ir * ir;
  col[3 * i] = r0 * ir3;
  col[3 * i + 1] = r1 * ir3;
  col[3 * i + 2] = r2 * ir3;
}

// T [n x m] = A^T, A [m x n] column-major
__global__ void k_fmm_transpose_rect(const double* __restrict__ A, int m, int n, double* __restrict__ T) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  if (i < m) T[(size_t)i * n + j] = A[(size_t)j * m + i];
}

__global__ void k_fmm_transpose(const double* __restrict__ A, int n, double* __restrict__ T) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  if (i < n) T[(size_t)i * n + j] = A[(size_t)j * n + i];
}

static int fgrid(size_t work) { return (int)std::max<size_t>(1, std::min<size_t>((work + 255) / 256, 8192)); }

__global__ void k_fmm_eye(double* R, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) R[(size_t)i * n + i] = 1.0;
}

__global__ void k_fmm_axpy(double* y, const double* x, size_t n) {
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) y[e] += x[e];
}

__global__ void k_fmm_tikhonov(double* G, int n, double eps) {
  __shared__ double mx;
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int i = 0; i < n; ++i) m = fmax(m, G[(size_t)i * n + i]);
    mx = m;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) G[(size_t)i * n + i] += eps * mx;
}

// sorted source records {y, n, f~ = cS w f, q~ = cD w q}
__global__ void k_fmm_records(int N, const int* __restrict__ perm, const double* __restrict__ src,
                              const double* __restrict__ sigS, const double* __restrict__ sigD, double cS, double cD,
                              double* __restrict__ rec) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= N) return;
  const int i = perm[k];
  const double* s = src + 8 * (size_t)i;
  double* o = rec + 12 * (size_t)k;
  o[0] = s[0]; o[1] = s[1]; o[2] = s[2];
  o[3] = s[4]; o[4] = s[5]; o[5] = s[6];
  const double w = s[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    o[6 + c] = sigS ? cS * w * sigS[3 * (size_t)i + c] : 0.0;
    o[9 + c] = sigD ? cD * w * sigD[3 * (size_t)i + c] : 0.0;
  }
}

// the K1 pair kernel, one direction: source record s at y -> target x
__device__ __forceinline__ void fmm_pair(double x0, double x1, double x2, const double* s, bool doS, bool doD,
                                         double& u0, double& u1, double& u2) {
  const double r0 = x0 - s[0], r1 = x1 - s[1], r2 = x2 - s[2];
  const double rr = fma(r2, r2, fma(r1, r1, r0 * r0));
  const double ir = rsqrt(rr), ir2 = ir * ir, ir3 = ir * ir2;
  double t = 0.0;
  if (doD) {
    const double rn = fma(r2, s[5], fma(r1, s[4], r0 * s[3]));
    const double rq = fma(r2, s[11], fma(r1, s[10], r0 * s[9]));
    t = rn * rq * ir3 * ir2;
  }
  if (doS) {
    const double rf = fma(r2, s[8], fma(r1, s[7], r0 * s[6]));
    t = fma(rf, ir3, t);
    u0 = fma(s[6], ir, u0);
    u1 = fma(s[7], ir, u1);
    u2 = fma(s[8], ir, u2);
  }
  u0 = fma(r0, t, u0);
  u1 = fma(r1, t, u1);
  u2 = fma(r2, t, u2);
}

// P2M: upward check potential of every occupied leaf at its check surface (2.95 r around the centre)
__global__ void __launch_bounds__(128) k_fmm_p2m(const double* __restrict__ rec, const int* __restrict__ start,
                                                 const double* __restrict__ surf, int ns, const double* __restrict__ ctr,
                                                 double rad, bool doS, bool doD, double* __restrict__ uck) {
  __shared__ double sr[128 * 12];
  const int b = blockIdx.x, s0 = start[b], s1 = start[b + 1];
  const double c0 = ctr[3 * b], c1 = ctr[3 * b + 1], c2 = ctr[3 * b + 2];
  for (int k0 = 0; k0 < ns; k0 += 128) {
    const int k = k0 + threadIdx.x;
    double x0 = 0, x1 = 0, x2 = 0, u0 = 0, u1 = 0, u2 = 0;
    if (k < ns) {
      x0 = c0 + rad * surf[3 * k];
      x1 = c1 + rad * surf[3 * k + 1];
      x2 = c2 + rad * surf[3 * k + 2];
    }
    for (int j0 = s0; j0 < s1; j0 += 128) {
      const int nj = min(128, s1 - j0);
      __syncthreads();
      for (int e = threadIdx.x; e < nj * 12; e += 128) sr[e] = rec[12 * (size_t)j0 + e];
      __syncthreads();
      if (k < ns)
        for (int j = 0; j < nj; ++j) fmm_pair(x0, x1, x2, sr + 12 * j, doS, doD, u0, u1, u2);
    }
    if (k < ns) {
      double* o = uck + (size_t)b * 3 * ns + 3 * k;
      o[0] = u0; o[1] = u1; o[2] = u2;
    }
  }
}

// The K1 pair kernel with K1's rsqrt (one MUFU.RSQ64H seed + the series to e^2, |e| <= 2^-19; allpairs.cu);
// rho = 0 (the target itself) contributes nothing
__device__ __forceinline__ double fmm_seed(double rr) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(rr));
  return rr > 0.0 ? y : 0.0;
}
template <int MODE>
__device__ __forceinline__ void fmm_pair_fast(double x0, double x1, double x2, const double* s, double& u0,
                                              double& u1, double& u2) {
  const double r0 = x0 - s[0], r1 = x1 - s[1], r2 = x2 - s[2];
  const double rr = fma(r2, r2, fma(r1, r1, r0 * r0));
  const double y = fmm_seed(rr), y2 = y * y;
  const double e = fma(-rr, y2, 1.0);
  double t;
  if (MODE == MODE_D) {
    const double s5 = (y * (y2 * y2)) * fma(e, fma(e, 4.375, 2.5), 1.0);
    const double rn = fma(r2, s[5], fma(r1, s[4], r0 * s[3]));
    const double rq = fma(r2, s[11], fma(r1, s[10], r0 * s[9]));
    t = (rn * rq) * s5;
  } else {
    const double sv = fma(y * e, fma(e, 0.375, 0.5), y);
    const double s2 = sv * sv, s3 = s2 * sv;
    const double rf = fma(r2, s[8], fma(r1, s[7], r0 * s[6]));
    t = rf * s3;
    if (MODE == MODE_SD) {
      const double rn = fma(r2, s[5], fma(r1, s[4], r0 * s[3]));
      const double rq = fma(r2, s[11], fma(r1, s[10], r0 * s[9]));
      t = fma(rn * rq, s3 * s2, t);
    }
    u0 = fma(s[6], sv, u0);
    u1 = fma(s[7], sv, u1);
    u2 = fma(s[8], sv, u2);
  }
  u0 = fma(r0, t, u0);
  u1 = fma(r1, t, u1);
  u2 = fma(r2, t, u2);
}

// Leaves: near field (27 neighbour leaves) + L2P from the leaf's downward equivalent density; two targets per
// thread share every staged source; writes out[node] in the original order
constexpr int FL_T = 64;
template <int MODE, int FL_R>
__global__ void __launch_bounds__(FL_T) k_fmm_leaf(const double* __restrict__ rec, const int* __restrict__ start,
                                                   const int* __restrict__ nbr, const int* __restrict__ perm,
                                                   const double* __restrict__ surf, int ns,
                                                   const double* __restrict__ ctr, double rad,
                                                   const double* __restrict__ deq, double* __restrict__ out) {
  __shared__ __align__(16) double sr[FL_T * 12];
  const int b = blockIdx.x, t0 = start[b], t1 = start[b + 1];
  int k[FL_R];
  double x[FL_R][3], u[FL_R][3];
#pragma unroll
  for (int r = 0; r < FL_R; ++r) {
    k[r] = t0 + blockIdx.y * FL_T * FL_R + r * FL_T + threadIdx.x;
    const int kk = min(k[r], t1 - 1);  // inactive lanes compute a duplicate and do not store
    x[r][0] = rec[12 * (size_t)kk];
    x[r][1] = rec[12 * (size_t)kk + 1];
    x[r][2] = rec[12 * (size_t)kk + 2];
    u[r][0] = u[r][1] = u[r][2] = 0.0;
  }
  if (t0 + blockIdx.y * FL_T * FL_R >= t1) return;
  for (int q = 0; q < 27; ++q) {
    const int nb = nbr[27 * b + q];
    if (nb < 0) continue;
    const int s0 = start[nb], s1 = start[nb + 1];
    for (int j0 = s0; j0 < s1; j0 += FL_T) {
      const int nj = min(FL_T, s1 - j0);
      __syncthreads();
      for (int e = threadIdx.x; e < nj * 12; e += FL_T) sr[e] = rec[12 * (size_t)j0 + e];
      __syncthreads();
#pragma unroll 2
      for (int j = 0; j < nj; ++j)
#pragma unroll
        for (int r = 0; r < FL_R; ++r) fmm_pair_fast<MODE>(x[r][0], x[r][1], x[r][2], sr + 12 * j, u[r][0], u[r][1], u[r][2]);
    }
  }
  // L2P: Stokeslet equivalent density on the downward equivalent surface (2.95 r)
  const double c0 = ctr[3 * b], c1 = ctr[3 * b + 1], c2 = ctr[3 * b + 2];
  const double* ph = deq + (size_t)b * 3 * ns;
  for (int j0 = 0; j0 < ns; j0 += FL_T) {
    const int nj = min(FL_T, ns - j0);
    __syncthreads();
    for (int e = threadIdx.x; e < nj; e += FL_T) {
      const int j = j0 + e;
      sr[6 * e] = c0 + rad * surf[3 * j];
      sr[6 * e + 1] = c1 + rad * surf[3 * j + 1];
      sr[6 * e + 2] = c2 + rad * surf[3 * j + 2];
      sr[6 * e + 3] = ph[3 * j];
      sr[6 * e + 4] = ph[3 * j + 1];
      sr[6 * e + 5] = ph[3 * j + 2];
    }
    __syncthreads();
    for (int j = 0; j < nj; ++j) {
      const double* sp = sr + 6 * j;
#pragma unroll
      for (int r = 0; r < FL_R; ++r) {
        const double r0 = x[r][0] - sp[0], r1 = x[r][1] - sp[1], r2 = x[r][2] - sp[2];
        const double rr = fma(r2, r2, fma(r1, r1, r0 * r0));
        const double ir = rsqrt(rr), ir3 = ir * ir * ir;
        const double t = fma(r2, sp[5], fma(r1, sp[4], r0 * sp[3])) * ir3;
        u[r][0] = fma(sp[3], ir, fma(r0, t, u[r][0]));
        u[r][1] = fma(sp[4], ir, fma(r1, t, u[r][1]));
        u[r][2] = fma(sp[5], ir, fma(r2, t, u[r][2]));
      }
    }
  }
#pragma unroll
  for (int r = 0; r < FL_R; ++r)
    if (k[r] < t1) {
      const int i = perm[k[r]];
      out[3 * (size_t)i] = u[r][0];
      out[3 * (size_t)i + 1] = u[r][1];
      out[3 * (size_t)i + 2] = u[r][2];
    }
}

// Small leaves (c4 at order 6: ~230 points per leaf).  One CTA per (leaf, 64-target chunk) leaves the SMs
// unevenly loaded: a corner leaf sees 8 neighbour leaves, an interior one 27, the whole grid is resident at once
// and the kernel ends with the most loaded SM (ncu, profiles/r02_fmm_leaf_seg.md: FP64 pipe 37-64 % of the
// elapsed time from SM to SM).  Here the concatenated source list of a leaf's neighbours is cut into segments of
// about FMM_SEG sources, so every CTA (leaf, chunk, segment) costs about the same and the SMs stay full to the
// end; segment K_b of a leaf is its L2P.  Each CTA stores its partial sum, k_fmm_leaf_sum adds a target's
// partials in segment order (a fixed order: bit-reproducible) and writes out[node] in the original order.
template <int MODE, bool SELF, int UNR>
__device__ __forceinline__ void fmm_leaf_chunk(const double* __restrict__ sr, int nj, double x0, double x1, double x2,
                                               double& u0, double& u1, double& u2) {
#pragma unroll UNR
  for (int j = 0; j < nj; ++j) {
    const double* s = sr + 12 * j;
    const double r0 = x0 - s[0], r1 = x1 - s[1], r2 = x2 - s[2];
    const double rr = fma(r2, r2, fma(r1, r1, r0 * r0));
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(rr));
    if (SELF) y = __double2hiint(rr) != 0 || __double2loint(rr) != 0 ? y : 0.0;  // rho = 0: the target itself
    const double y2 = y * y;
    const double e = fma(-rr, y2, 1.0);
    double t;
    if (MODE == MODE_D) {
      const double s5 = (y * (y2 * y2)) * fma(e, fma(e, 4.375, 2.5), 1.0);
      const double rn = fma(r2, s[5], fma(r1, s[4], r0 * s[3]));
      const double rq = fma(r2, s[11], fma(r1, s[10], r0 * s[9]));
      t = (rn * rq) * s5;
    } else {
      const double sv = fma(y * e, fma(e, 0.375, 0.5), y);
      const double s2 = sv * sv, s3 = s2 * sv;
      const double rf = fma(r2, s[8], fma(r1, s[7], r0 * s[6]));
      t = rf * s3;
      if (MODE == MODE_SD) {
        const double rn = fma(r2, s[5], fma(r1, s[4], r0 * s[3]));
        const double rq = fma(r2, s[11], fma(r1, s[10], r0 * s[9]));
        t = fma(rn * rq, s3 * s2, t);
      }
      u0 = fma(s[6], sv, u0);
      u1 = fma(s[7], sv, u1);
      u2 = fma(s[8], sv, u2);
    }
    u0 = fma(r0, t, u0);
    u1 = fma(r1, t, u1);
    u2 = fma(r2, t, u2);
  }
}

template <int MODE, int UNR>
__global__ void __launch_bounds__(FL_T) k_fmm_leaf_seg(const int4* __restrict__ items, const double* __restrict__ rec,
                                                       const int* __restrict__ start, const int* __restrict__ nbr,
                                                       const double* __restrict__ surf, int ns,
                                                       const double* __restrict__ ctr, double rad,
                                                       const double* __restrict__ deq, int N,
                                                       double* __restrict__ part) {
  __shared__ __align__(16) double sr[FL_T * 12];
  const int4 it = items[blockIdx.x];
  const int b = it.x, seg = it.z, seglen = it.w;
  const int t0 = start[b], t1 = start[b + 1];
  const int k = t0 + it.y * FL_T + threadIdx.x;
  const int kk = min(k, t1 - 1);  // inactive lanes compute a duplicate and do not store
  // a warp without any target (the chunk's tail) only helps staging: it keeps off the FP64 pipe
  const bool warp_on = t0 + it.y * FL_T + (int)(threadIdx.x & ~31u) < t1;
  const double x0 = rec[12 * (size_t)kk], x1 = rec[12 * (size_t)kk + 1], x2 = rec[12 * (size_t)kk + 2];
  double u0 = 0.0, u1 = 0.0, u2 = 0.0;
  if (seglen > 0) {  // near field: sources [lo, hi) of the concatenated neighbour leaves
    const int lo = seg * seglen, hi = lo + seglen;
    int off = 0;
    for (int q = 0; q < 27 && off < hi; ++q) {
      const int nb = nbr[27 * b + q];
      if (nb < 0) continue;
      const int s0 = start[nb], cnt = start[nb + 1] - s0;
      const int a = max(lo - off, 0), e = min(hi - off, cnt);
      off += cnt;
      for (int j0 = s0 + a; j0 < s0 + e; j0 += FL_T) {
        const int nj = min(FL_T, s0 + e - j0);
        __syncthreads();
        {
          const double2* g2 = reinterpret_cast<const double2*>(rec + 12 * (size_t)j0);
          double2* s2 = reinterpret_cast<double2*>(sr);
          for (int w = threadIdx.x; w < nj * 6; w += FL_T) s2[w] = g2[w];
        }
        __syncthreads();
        if (!warp_on) continue;
        if (nb == b) fmm_leaf_chunk<MODE, true, UNR>(sr, nj, x0, x1, x2, u0, u1, u2);
        else fmm_leaf_chunk<MODE, false, UNR>(sr, nj, x0, x1, x2, u0, u1, u2);
      }
    }
  } else {  // L2P: Stokeslet equivalent density on the downward equivalent surface (2.95 r)
    const double c0 = ctr[3 * b], c1 = ctr[3 * b + 1], c2 = ctr[3 * b + 2];
    const double* ph = deq + (size_t)b * 3 * ns;
    for (int j0 = 0; j0 < ns; j0 += FL_T) {
      const int nj = min(FL_T, ns - j0);
      __syncthreads();
      for (int e = threadIdx.x; e < nj; e += FL_T) {
        const int j = j0 + e;
        sr[6 * e] = c0 + rad * surf[3 * j];
        sr[6 * e + 1] = c1 + rad * surf[3 * j + 1];
        sr[6 * e + 2] = c2 + rad * surf[3 * j + 2];
        sr[6 * e + 3] = ph[3 * j];
        sr[6 * e + 4] = ph[3 * j + 1];
        sr[6 * e + 5] = ph[3 * j + 2];
      }
      __syncthreads();
      if (!warp_on) continue;
#pragma unroll 2
      for (int j = 0; j < nj; ++j) {
        const double* sp = sr + 6 * j;
        const double r0 = x0 - sp[0], r1 = x1 - sp[1], r2 = x2 - sp[2];
        const double rr = fma(r2, r2, fma(r1, r1, r0 * r0));
        double y;  // the surface lies outside the leaf: rho > 0
        asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(rr));
        const double e = fma(-rr, y * y, 1.0);
        const double ir = fma(y * e, fma(e, 0.375, 0.5), y), ir3 = ir * ir * ir;
        const double t = fma(r2, sp[5], fma(r1, sp[4], r0 * sp[3])) * ir3;
        u0 = fma(sp[3], ir, fma(r0, t, u0));
        u1 = fma(sp[4], ir, fma(r1, t, u1));
        u2 = fma(sp[5], ir, fma(r2, t, u2));
      }
    }
  }
  if (k < t1) {
    double* o = part + ((size_t)seg * N + k) * 3;
    o[0] = u0;
    o[1] = u1;
    o[2] = u2;
  }
}

__global__ void k_fmm_leaf_sum(int N, const int* __restrict__ tparts, const int* __restrict__ perm,
                               const double* __restrict__ part, double* __restrict__ out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= N) return;
  const int np = tparts[k];
  double u0 = 0.0, u1 = 0.0, u2 = 0.0;
  for (int s = 0; s < np; ++s) {
    const double* o = part + ((size_t)s * N + k) * 3;
    u0 += o[0];
    u1 += o[1];
    u2 += o[2];
  }
  const int i = perm[k];
  out[3 * (size_t)i] = u0;
  out[3 * (size_t)i + 1] = u1;
  out[3 * (size_t)i + 2] = u2;
}

// dst[:, j] = src[:, idx[j]] (columns of length m)
__global__ void k_fmm_gather(const double* __restrict__ src, int m, const int* __restrict__ idx, int cnt,
                             double* __restrict__ dst) {
  const size_t tot = (size_t)m * cnt;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (size_t)gridDim.x * blockDim.x) {
    const int j = (int)(e / m), r = (int)(e % m);
    dst[e] = src[(size_t)idx[j] * m + r];
  }
}

// dst[:, idx[j]] += src[:, j]  (idx distinct within one call)
__global__ void k_fmm_scatter_add(double* __restrict__ dst, int m, const int* __restrict__ idx, int cnt,
                                  const double* __restrict__ src) {
  const size_t tot = (size_t)m * cnt;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (size_t)gridDim.x * blockDim.x) {
    const int j = (int)(e / m), r = (int)(e % m);
    dst[(size_t)idx[j] * m + r] += src[e];
  }
}

// dck[:, t] += sum over t's M2L pairs (offset order) of C[:, pos]
__global__ void k_fmm_m2l_reduce(double* __restrict__ dck, int m, int nt, const int* __restrict__ ptr,
                                 const int* __restrict__ pos, const double* __restrict__ C) {
  const size_t tot = (size_t)m * nt;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (size_t)gridDim.x * blockDim.x) {
    const int t = (int)(e / m), r = (int)(e % m);
    double v = dck[e];
    for (int k = ptr[t]; k < ptr[t + 1]; ++k) v += C[(size_t)pos[k] * m + r];
    dck[e] = v;
  }
}


// ------------------------------------------------------------------ operators (unit box)
// pinv of K (mr x nc, column-major): (K^T K + eps max diag I)^-1 K^T into P [nc x mr]
static void fmm_pinv(const double* K, int mr, int nc, double* P, cudaStream_t st) {
  DBuf<double> G;
  G.alloc((size_t)nc * nc);
  blas_dgemm(st, FMM_OP_T, FMM_OP_N, nc, nc, mr, 1.0, K, mr, K, mr, 0.0, G.p, nc);
  double eps = 1e-13;
  if (const char* e = getenv("BPQN_FMM_EPS")) eps = atof(e);  // studies (profiles/r02_fmm.md)
  k_fmm_tikhonov<<<1, 256, 0, st>>>(G.p, nc, eps);
  BPQN_CHECK_LAUNCH();
  dev_potrf(st, G.p, nc, nc);
  k_fmm_transpose_rect<<<dim3((mr + 255) / 256, nc), 256, 0, st>>>(K, mr, nc, P);
  BPQN_CHECK_LAUNCH();
  blas_dtrsm(st, 0, 0, nc, mr, G.p, nc, P, nc);
  blas_dtrsm(st, 0, 1, nc, mr, G.p, nc, P, nc);
  // iterated Tikhonov: P += (K^T K + eps I)^-1 K^T (I - K P), which lifts the regularisation's damping of the
  // small singular directions by another factor eps / (sigma^2 + eps) per step
  int refine = 2;
  if (const char* e = getenv("BPQN_FMM_REFINE")) refine = atoi(e);
  if (refine > 0) {
    DBuf<double> R, D;
    R.alloc((size_t)mr * mr);
    D.alloc((size_t)nc * mr);
    for (int it = 0; it < refine; ++it) {
      BPQN_CUDA(cudaMemsetAsync(R.p, 0, 8 * (size_t)mr * mr, st));
      k_fmm_eye<<<(mr + 255) / 256, 256, 0, st>>>(R.p, mr);
      BPQN_CHECK_LAUNCH();
      blas_dgemm(st, FMM_OP_N, FMM_OP_N, mr, mr, nc, -1.0, K, mr, P, nc, 1.0, R.p, mr);   // I - K P
      blas_dgemm(st, FMM_OP_T, FMM_OP_N, nc, mr, mr, 1.0, K, mr, R.p, mr, 0.0, D.p, nc);  // K^T (I - K P)
      blas_dtrsm(st, 0, 0, nc, mr, G.p, nc, D.p, nc);
      blas_dtrsm(st, 0, 1, nc, mr, G.p, nc, D.p, nc);
      k_fmm_axpy<<<fgrid((size_t)nc * mr), 256, 0, st>>>(P, D.p, (size_t)nc * mr);
      BPQN_CHECK_LAUNCH();
    }
  }
  BPQN_CUDA(cudaStreamSynchronize(st));
}

// Stokeslet block G(x_i <- y_j) with x = sx surf + ox (rows), y = sy surf + oy (columns), ld = 3 ns; with
// src_fac != 0 one more column: the point source at oy with factor src_fac (upward equivalents)
static void fmm_gmat(const Fmm& F, double sx, double3 ox, double sy, double3 oy, double* K, cudaStream_t st,
                     double src_fac = 0.0) {
  const int n = F.ns;
  k_fmm_gmat<<<dim3((n + 127) / 128, n), 128, 0, st>>>(F.surf.p, n, sx, ox, F.surf.p, n, sy, oy, K, 3 * n);
  BPQN_CHECK_LAUNCH();
  if (src_fac != 0.0) {
    k_fmm_srccol<<<(n + 127) / 128, 128, 0, st>>>(F.surf.p, n, sx, ox, oy, src_fac, K + (size_t)3 * n * 3 * n);
    BPQN_CHECK_LAUNCH();
  }
}

// Unit box (half-width 1).  Upward equivalents carry 3 ns Stokeslet densities plus one point source at the box
// centre, whose kernel is scaled by the box half-width (r (x - y) / |x - y|^3) so that every operator stays
// homogeneous of degree -1 and scales by 1 / r per level like the Stokeslet.
// Pivoted Cholesky of the n x n Gram matrix G (column-major, symmetric PSD) down to a residual diagonal of
// tol^2 max diag: the pivots I (r of them) and the interpolation matrix W [n][r] (column-major) with
// rows(A) ~ W rows_I(A) for the A behind G = A A^T (W[I, :] = identity).
static int fmm_pivchol_interp(const std::vector<double>& G, int n, double tol, int rmax, std::vector<int>& I,
                              std::vector<double>& W) {
  std::vector<double> d(n), Lm;  // Lm [n][r] column-major, grown column by column
  double d0 = 0.0;
  for (int i = 0; i < n; ++i) {
    d[i] = G[(size_t)i * n + i];
    d0 = std::max(d0, d[i]);
  }
  std::vector<char> used(n, 0);
  I.clear();
  int r = 0;
  while (r < rmax) {
    int pv = -1;
    double best = tol * tol * d0;
    for (int i = 0; i < n; ++i)
      if (!used[i] && d[i] > best) {
        best = d[i];
        pv = i;
      }
    if (pv < 0) break;
    Lm.resize((size_t)n * (r + 1));
    double* col = Lm.data() + (size_t)n * r;
    for (int i = 0; i < n; ++i) col[i] = G[(size_t)pv * n + i];
    for (int j = 0; j < r; ++j) {
      const double* cj = Lm.data() + (size_t)n * j;
      const double f = cj[pv];
      for (int i = 0; i < n; ++i) col[i] -= cj[i] * f;
    }
    const double piv = std::sqrt(std::max(col[pv], 1e-300));
    for (int i = 0; i < n; ++i) {
      col[i] = used[i] ? 0.0 : col[i] / piv;
      d[i] -= col[i] * col[i];
    }
    used[pv] = 1;
    d[pv] = 0.0;
    I.push_back(pv);
    ++r;
  }
  // W L_I = L with L_I = L[I, :] lower triangular (L[I[k], j] = 0 for j > k): back substitution row by row
  W.assign((size_t)n * r, 0.0);
  std::vector<double> w(r);
  for (int i = 0; i < n; ++i) {
    if (used[i]) continue;
    for (int k = r - 1; k >= 0; --k) {
      double v = Lm[(size_t)n * k + i];
      for (int j = k + 1; j < r; ++j) v -= w[j] * Lm[(size_t)n * k + I[j]];
      w[k] = v / Lm[(size_t)n * k + I[k]];
    }
    for (int k = 0; k < r; ++k) W[(size_t)n * k + i] = w[k];
  }
  for (int k = 0; k < r; ++k) W[(size_t)n * k + I[k]] = 1.0;
  return r;
}

// Mc[o][a + rU b] = M[o][I[a] + m J[b]]
__global__ void k_fmm_m2l_core(const double* __restrict__ M, int m, int mu, const int* __restrict__ I, int rU,
                               const int* __restrict__ J, int rV, double* __restrict__ Mc) {
  const size_t o = blockIdx.y;
  const int tot = rU * rV;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += gridDim.x * blockDim.x) {
    const int a = e % rU, b = e / rU;
    Mc[o * tot + e] = M[o * (size_t)m * mu + I[a] + (size_t)m * J[b]];
  }
}

// Shared row / column skeletons of the 316 M2L matrices (order <= 8: the low orders of the FMM-accelerated
// refinement, whose Krylov steps tolerate 1e-4).  The rows of [M2L_1 ... M2L_316] and the columns of
// [M2L_1; ...; M2L_316] are numerically dependent to tol, so M2L_o ~ WU M2L_o[I, J] WV^T: the per-pair GEMM
// shrinks from 3ns x (3ns + 1) to rU x rV, with one WV^T / WU GEMM per level around it.
static void fmm_compress_m2l(Fmm& F, cudaStream_t st) {
  F.m2l_comp = false;
  // default tolerance: about the order's own far-field error (D layer, c4: order 5 2e-3, 6 1.4e-4, 7 1.6e-5,
  // 8 2.4e-6), so the compressed FMM stays within ~1.5x of it (order 6: 2.0e-4; profiles/r02_fmm_m2l.md);
  // orders <= 4 have nothing to gain (full rank at 1e-3), orders >= 9 are used for accuracy and stay exact
  double tol = F.pe == 5 ? 1e-3 : F.pe == 6 ? 1e-4 : F.pe == 7 ? 1e-5 : F.pe == 8 ? 2e-6 : 0.0;
  if (const char* e = getenv("BPQN_FMM_M2L_TOL")) tol = atof(e);  // 0: off
  if (!(tol > 0.0) || F.pe > 8) return;
  const int m = 3 * F.ns, mu = m + 1;
  const size_t mmu = (size_t)m * mu;
  DBuf<double> GU, GV;
  GU.alloc((size_t)m * m);
  GV.alloc((size_t)mu * mu);
  for (int o = 0; o < FMM_NOFF; ++o) {  // (one GEMM over the 316 mu columns overflows nothing but is no faster)
    blas_dgemm(st, FMM_OP_N, FMM_OP_T, m, m, mu, 1.0, F.M2L.p + o * mmu, m, F.M2L.p + o * mmu, m, o ? 1.0 : 0.0,
               GU.p, m);
    blas_dgemm(st, FMM_OP_T, FMM_OP_N, mu, mu, m, 1.0, F.M2L.p + o * mmu, m, F.M2L.p + o * mmu, m, o ? 1.0 : 0.0,
               GV.p, mu);
  }
  std::vector<double> hU((size_t)m * m), hV((size_t)mu * mu);
  BPQN_CUDA(cudaMemcpyAsync(hU.data(), GU.p, 8 * hU.size(), cudaMemcpyDeviceToHost, st));
  BPQN_CUDA(cudaMemcpyAsync(hV.data(), GV.p, 8 * hV.size(), cudaMemcpyDeviceToHost, st));
  BPQN_CUDA(cudaStreamSynchronize(st));
  std::vector<int> I, J;
  std::vector<double> WU, WV;
  const int rU = fmm_pivchol_interp(hU, m, tol, m, I, WU);
  const int rV = fmm_pivchol_interp(hV, mu, tol, mu, J, WV);
  if (getenv("BPQN_FMM_DEBUG")) fprintf(stderr, "[bpqn fmm] M2L skeletons: %d of %d rows, %d of %d columns (tol %.1e)\n", rU, m, rV, mu, tol);
  if ((double)rU * rV > 0.5 * (double)m * mu || rU < 8 || rV < 8) return;  // not worth the two extra GEMMs
  F.rU = rU;
  F.rV = rV;
  fmm_upload(F.WU, WU, st);
  fmm_upload(F.WV, WV, st);
  DBuf<int> dI, dJ;
  fmm_upload(dI, I, st);
  fmm_upload(dJ, J, st);
  F.M2Lc.alloc((size_t)FMM_NOFF * rU * rV);
  k_fmm_m2l_core<<<dim3((rU * rV + 255) / 256, FMM_NOFF), 256, 0, st>>>(F.M2L.p, m, mu, dI.p, rU, dJ.p, rV, F.M2Lc.p);
  BPQN_CHECK_LAUNCH();
  BPQN_CUDA(cudaStreamSynchronize(st));
  F.m2l_comp = true;
}

static void fmm_operators(Fmm& F, cudaStream_t st) {
  const int pe = F.pe;
  std::vector<double> s;
  for (int i = 0; i < pe; ++i)
    for (int j = 0; j < pe; ++j)
      for (int k = 0; k < pe; ++k) {
        if (!(i == 0 || i == pe - 1 || j == 0 || j == pe - 1 || k == 0 || k == pe - 1)) continue;
        s.push_back(-1.0 + 2.0 * i / (pe - 1));
        s.push_back(-1.0 + 2.0 * j / (pe - 1));
        s.push_back(-1.0 + 2.0 * k / (pe - 1));
      }
  F.ns = (int)(s.size() / 3);
  F.surf.alloc(s.size());
  BPQN_CUDA(cudaMemcpyAsync(F.surf.p, s.data(), 8 * s.size(), cudaMemcpyHostToDevice, st));
  const int m = 3 * F.ns, mu = m + 1;
  const size_t mm = (size_t)m * m, mmu = (size_t)m * mu;
  const double3 z{0, 0, 0};
  DBuf<double> K;
  K.alloc(mmu);
  F.UC2E.alloc(mmu);
  F.DC2E.alloc(mm);
  fmm_gmat(F, FMM_OUT, z, FMM_IN, z, K.p, st, 1.0);  // upward check <- upward equivalent (+ source)
  fmm_pinv(K.p, m, mu, F.UC2E.p, st);
  fmm_gmat(F, FMM_IN, z, FMM_OUT, z, K.p, st);       // downward check <- downward equivalent
  fmm_pinv(K.p, m, m, F.DC2E.p, st);
  F.M2M.alloc(8 * mmu);
  F.L2L.alloc(8 * mm);
  for (int c = 0; c < 8; ++c) {
    const double3 cc{(c & 4) ? 0.5 : -0.5, (c & 2) ? 0.5 : -0.5, (c & 1) ? 0.5 : -0.5};
    fmm_gmat(F, FMM_OUT, z, 0.5 * FMM_IN, cc, F.M2M.p + c * mmu, st, 0.5);  // parent up-check <- child up-equiv
    fmm_gmat(F, 0.5 * FMM_IN, cc, FMM_OUT, z, F.L2L.p + c * mm, st);        // child down-check <- parent down-equiv
  }
  F.offs.clear();
  for (int a = -3; a <= 3; ++a)
    for (int b = -3; b <= 3; ++b)
      for (int c = -3; c <= 3; ++c)
        if (std::max(std::abs(a), std::max(std::abs(b), std::abs(c))) >= 2) {
          F.offs.push_back(a);
          F.offs.push_back(b);
          F.offs.push_back(c);
        }
  BPQN_REQUIRE((int)F.offs.size() == 3 * FMM_NOFF, "FMM offsets");
  F.M2L.alloc((size_t)FMM_NOFF * mmu);
  for (int o = 0; o < FMM_NOFF; ++o) {  // target at the origin, source box centre at 2 o
    const double3 so{2.0 * F.offs[3 * o], 2.0 * F.offs[3 * o + 1], 2.0 * F.offs[3 * o + 2]};
    fmm_gmat(F, FMM_IN, z, FMM_IN, so, F.M2L.p + o * mmu, st, 1.0);
  }
  BPQN_CUDA(cudaStreamSynchronize(st));
  fmm_compress_m2l(F, st);
  F.ops_ready = true;
}

// ------------------------------------------------------------------ tree (host lists)
void fmm_build(Geom& g, const std::vector<double>& X, cudaStream_t st) {
  if (g.fmm_order <= 0) return;
  BPQN_REQUIRE(g.fmm_order >= 3 && g.fmm_order <= 12, "fmm_order must be in [3, 12]");
  if (!g.fmm) g.fmm = new Fmm();
  Fmm& F = *g.fmm;
  if (!F.ops_ready) {
    F.pe = g.fmm_order;
    fmm_operators(F, st);
  }
  const int N = g.n;
  double mn[3] = {1e300, 1e300, 1e300}, mx[3] = {-1e300, -1e300, -1e300};
  for (int i = 0; i < N; ++i)
    for (int c = 0; c < 3; ++c) {
      mn[c] = std::min(mn[c], X[3 * (size_t)i + c]);
      mx[c] = std::max(mx[c], X[3 * (size_t)i + c]);
    }
  double ext = 0.0;
  for (int c = 0; c < 3; ++c) ext = std::max(ext, mx[c] - mn[c]);
  F.R0 = 0.5 * ext * (1.0 + 1e-9) + 1e-12;
  for (int c = 0; c < 3; ++c) F.lo[c] = 0.5 * (mn[c] + mx[c]) - F.R0;
  // leaf size balances the near field (~ points per leaf) against M2L (~ boxes x (p_e^3 - (p_e-2)^3)^2):
  // ~800 points per leaf at order 10, fewer at lower orders (c4 at order 6: 3 levels, 4.8 ms vs 15 ms at 2)
  const double leaf_pts = 800.0 * std::pow(F.pe / 10.0, 3);
  int L = std::max(2, (int)std::lround(std::log((double)N / leaf_pts) / std::log(8.0)));
  if (const char* e = getenv("BPQN_FMM_LEVELS")) L = std::max(2, atoi(e));
  L = std::min(L, 7);
  F.L = L;
  for (int l = 0; l < 8; ++l) F.lev[l].reset();
  // leaf box of every node, sorted order
  const int nL = 1 << L;
  std::vector<int> leafd(N);
  for (int i = 0; i < N; ++i) {
    int id[3];
    for (int c = 0; c < 3; ++c) {
      int v = (int)std::floor((X[3 * (size_t)i + c] - F.lo[c]) / (2.0 * F.R0) * nL);
      id[c] = std::min(nL - 1, std::max(0, v));
    }
    leafd[i] = (id[0] * nL + id[1]) * nL + id[2];
  }
  std::vector<int> perm(N);
  for (int i = 0; i < N; ++i) perm[i] = i;
  std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) { return leafd[a] < leafd[b]; });
  // occupancy per level (dense -> compact maps)
  std::vector<std::vector<int>> cmap(L + 1);
  for (int l = 0; l <= L; ++l) cmap[l].assign((size_t)1 << (3 * l), -1);
  auto coarsen = [&](int d, int from, int to) {  // dense index at level `from` -> its ancestor at `to`
    const int n = 1 << from, sh = from - to;
    const int x = d / (n * n), y = (d / n) % n, z = d % n;
    const int m = 1 << to;
    return (((x >> sh) * m) + (y >> sh)) * m + (z >> sh);
  };
  for (int k = 0; k < N; ++k) {
    const int d = leafd[perm[k]];
    for (int l = L; l >= 0; --l) {
      const int dl = coarsen(d, L, l);
      if (cmap[l][dl] < 0) {
        cmap[l][dl] = (int)F.lev[l].dense.size();
        F.lev[l].dense.push_back(dl);
      }
    }
  }
  // compact ids must follow the dense order at the leaf level for the point ranges: leaves were added in
  // sorted (dense) order; other levels are only used through the maps
  for (int l = 0; l <= L; ++l) {
    FmmLevel& V = F.lev[l];
    V.nocc = (int)V.dense.size();
    V.r = F.R0 / (1 << l);
    const int n = 1 << l;
    std::vector<double> ctr(3 * (size_t)V.nocc);
    for (int b = 0; b < V.nocc; ++b) {
      const int d = V.dense[b], x = d / (n * n), y = (d / n) % n, z = d % n;
      ctr[3 * b] = F.lo[0] + (2 * x + 1) * V.r;
      ctr[3 * b + 1] = F.lo[1] + (2 * y + 1) * V.r;
      ctr[3 * b + 2] = F.lo[2] + (2 * z + 1) * V.r;
    }
    fmm_upload(V.ctr, ctr, st);
    const size_t m = 3 * (size_t)F.ns * std::max(V.nocc, 1);
    V.ueq.alloc(m + std::max(V.nocc, 1));
    V.uck.alloc(m);
    V.deq.alloc(m);
    V.dck.alloc(m);
  }
  // leaf point ranges and neighbour lists
  FmmLevel& LV = F.lev[L];
  std::vector<int> start(LV.nocc + 1, 0);
  for (int k = 0; k < N; ++k) start[cmap[L][leafd[perm[k]]] + 1]++;
  for (int b = 0; b < LV.nocc; ++b) start[b + 1] += start[b];
  std::vector<int> nbr(27 * (size_t)LV.nocc, -1);
  for (int b = 0; b < LV.nocc; ++b) {
    const int d = LV.dense[b], x = d / (nL * nL), y = (d / nL) % nL, z = d % nL;
    int q = 0;
    for (int a = -1; a <= 1; ++a)
      for (int bb = -1; bb <= 1; ++bb)
        for (int c = -1; c <= 1; ++c, ++q) {
          const int xx = x + a, yy = y + bb, zz = z + c;
          if (xx < 0 || yy < 0 || zz < 0 || xx >= nL || yy >= nL || zz >= nL) continue;
          nbr[27 * (size_t)b + q] = cmap[L][(xx * nL + yy) * nL + zz];
        }
  }
  int maxleaf = 0;
  for (int b = 0; b < LV.nocc; ++b) maxleaf = std::max(maxleaf, start[b + 1] - start[b]);
  g.fmm_max_leaf = maxleaf;
  fmm_upload(F.perm, perm, st);
  fmm_upload(F.leaf_start, start, st);
  fmm_upload(F.leaf_nbr, nbr, st);
  // small leaves: equal-cost (leaf, chunk, segment) items for k_fmm_leaf_seg (segment K_b = the leaf's L2P)
  F.n_items = F.kmax = 0;
  if (maxleaf < 3 * FL_T * 4) {
    int seg_target = 512;  // c4 at order 6: D apply 3.54 ms (1024: 3.59, 2048: 3.77, 256: 3.53; one CTA per (leaf, chunk): 4.46)
    if (const char* e = getenv("BPQN_FMM_SEG")) seg_target = std::max(FL_T, atoi(e));
    std::vector<int> items, l2p, tparts(N);
    for (int b = 0; b < LV.nocc; ++b) {
      const int nb_pts = start[b + 1] - start[b];
      long long tot = 0;
      for (int q = 0; q < 27; ++q) {
        const int nb = nbr[27 * (size_t)b + q];
        if (nb >= 0) tot += start[nb + 1] - start[nb];
      }
      int K = (int)std::max(1LL, (tot + seg_target / 2) / seg_target);
      const int seglen = (int)(((tot + K - 1) / K + FL_T - 1) / FL_T) * FL_T;
      K = (int)((tot + seglen - 1) / seglen);
      for (int c = 0; c * FL_T < nb_pts; ++c) {
        for (int sgi = 0; sgi < K; ++sgi) {
          items.push_back(b); items.push_back(c); items.push_back(sgi); items.push_back(seglen);
        }
        l2p.push_back(b); l2p.push_back(c); l2p.push_back(K); l2p.push_back(0);
      }
      for (int k = start[b]; k < start[b + 1]; ++k) tparts[k] = K + 1;
      F.kmax = std::max(F.kmax, K + 1);
    }
    F.n_near = (int)(items.size() / 4);
    items.insert(items.end(), l2p.begin(), l2p.end());
    F.n_items = (int)(items.size() / 4);
    fmm_upload(F.leaf_items, items, st);
    fmm_upload(F.tparts, tparts, st);
    F.part.alloc((size_t)F.kmax * N * 3);
  }
  F.rec.alloc(12 * (size_t)N);
  // M2M / L2L octant pairs (parent level l, children at l + 1)
  size_t maxcols = 0;
  for (int l = 2; l < L; ++l) {
    FmmLevel& P = F.lev[l];
    const int nc = 1 << (l + 1);
    std::vector<std::vector<int>> pp(8), cc(8);
    for (int b = 0; b < F.lev[l + 1].nocc; ++b) {
      const int d = F.lev[l + 1].dense[b], x = d / (nc * nc), y = (d / nc) % nc, z = d % nc;
      const int oct = ((x & 1) << 2) | ((y & 1) << 1) | (z & 1);
      pp[oct].push_back(cmap[l][coarsen(d, l + 1, l)]);
      cc[oct].push_back(b);
    }
    std::vector<int> par_all, ch_all;
    for (int o = 0; o < 8; ++o) {
      P.n_oct[o] = (int)pp[o].size();
      fmm_upload(P.oct_par[o], pp[o], st);
      fmm_upload(P.oct_ch[o], cc[o], st);
      maxcols = std::max(maxcols, pp[o].size());
      P.oct_start[o] = (int)par_all.size();
      par_all.insert(par_all.end(), pp[o].begin(), pp[o].end());
      ch_all.insert(ch_all.end(), cc[o].begin(), cc[o].end());
    }
    P.oct_start[8] = P.n_child = (int)par_all.size();
    std::vector<int> pptr(P.nocc + 1, 0), ppos(par_all.size());
    for (int j : par_all) pptr[j + 1]++;
    for (int b = 0; b < P.nocc; ++b) pptr[b + 1] += pptr[b];
    {
      std::vector<int> fill(pptr.begin(), pptr.end() - 1);
      for (int j = 0; j < (int)par_all.size(); ++j) ppos[fill[par_all[j]]++] = j;  // octant order per parent
    }
    fmm_upload(P.par_all, par_all, st);
    fmm_upload(P.ch_all, ch_all, st);
    fmm_upload(P.par_ptr, pptr, st);
    fmm_upload(P.par_pos, ppos, st);
  }
  // M2L pairs per level l >= 2 (source a child of a neighbour of the target's parent, not adjacent)
  for (int l = 2; l <= L; ++l) {
    FmmLevel& V = F.lev[l];
    const int n = 1 << l;
    std::vector<std::vector<std::pair<int, int>>> byoff(FMM_NOFF);  // (target, source)
    std::vector<int> offidx(343, -1);
    for (int o = 0; o < FMM_NOFF; ++o)
      offidx[((F.offs[3 * o] + 3) * 7 + F.offs[3 * o + 1] + 3) * 7 + F.offs[3 * o + 2] + 3] = o;
    for (int t = 0; t < V.nocc; ++t) {
      const int d = V.dense[t], x = d / (n * n), y = (d / n) % n, z = d % n;
      const int px = x >> 1, py = y >> 1, pz = z >> 1;
      for (int sx = 2 * (px - 1); sx <= 2 * (px + 1) + 1; ++sx)
        for (int sy = 2 * (py - 1); sy <= 2 * (py + 1) + 1; ++sy)
          for (int sz = 2 * (pz - 1); sz <= 2 * (pz + 1) + 1; ++sz) {
            if (sx < 0 || sy < 0 || sz < 0 || sx >= n || sy >= n || sz >= n) continue;
            const int ox = sx - x, oy = sy - y, oz = sz - z;
            if (std::max(std::abs(ox), std::max(std::abs(oy), std::abs(oz))) < 2) continue;
            const int s = cmap[l][(sx * n + sy) * n + sz];
            if (s < 0) continue;
            byoff[offidx[((ox + 3) * 7 + oy + 3) * 7 + oz + 3]].push_back({t, s});
          }
    }
    std::vector<int> src, ptr(V.nocc + 1, 0), pos;
    V.off_start.assign(FMM_NOFF + 1, 0);
    std::vector<std::vector<int>> per_t(V.nocc);
    for (int o = 0; o < FMM_NOFF; ++o) {
      V.off_start[o] = (int)src.size();
      for (auto& pr : byoff[o]) {
        per_t[pr.first].push_back((int)src.size());
        src.push_back(pr.second);
      }
    }
    V.off_start[FMM_NOFF] = (int)src.size();
    V.n_pairs = (int)src.size();
    for (int t = 0; t < V.nocc; ++t) {
      ptr[t + 1] = ptr[t] + (int)per_t[t].size();
      pos.insert(pos.end(), per_t[t].begin(), per_t[t].end());
    }
    fmm_upload(V.m2l_src, src, st);
    fmm_upload(V.tgt_ptr, ptr, st);
    fmm_upload(V.tgt_pos, pos, st);
    maxcols = std::max(maxcols, (size_t)V.n_pairs);
  }
  maxcols = std::max<size_t>(maxcols, 1);
  const size_t m = 3 * (size_t)F.ns + 1;
  if (F.buf_cols < maxcols) {
    F.bufB.alloc(m * maxcols);
    F.bufC.alloc(m * maxcols);
    F.buf_cols = maxcols;
  }
  // grouped-batched M2L: per level the non-empty offsets' GEMMs (pointers into the fixed buffers)
  {
    // (compressed M2L: the rU x rV cores instead of the 3ns x (3ns + 1) matrices)
    const int mm3 = F.m2l_comp ? F.rU : 3 * F.ns, muu = F.m2l_comp ? F.rV : 3 * F.ns + 1;
    const double* m2l = F.m2l_comp ? F.M2Lc.p : F.M2L.p;
    for (int l = 2; l <= L; ++l) {
      FmmLevel& V = F.lev[l];
      V.g_m.clear(); V.g_n.clear(); V.g_k.clear(); V.g_lda.clear(); V.g_ldb.clear(); V.g_ldc.clear();
      V.g_alpha.clear();
      std::vector<const double*> pa, pb;
      std::vector<double*> pc;
      for (int o = 0; o < FMM_NOFF; ++o) {
        const int c0 = V.off_start[o], cnt = V.off_start[o + 1] - c0;
        if (!cnt) continue;
        V.g_m.push_back(mm3); V.g_n.push_back(cnt); V.g_k.push_back(muu);
        V.g_lda.push_back(mm3); V.g_ldb.push_back(muu); V.g_ldc.push_back(mm3);
        V.g_alpha.push_back(1.0 / V.r);
        pa.push_back(m2l + (size_t)o * mm3 * muu);
        pb.push_back(F.bufB.p + (size_t)c0 * muu);
        pc.push_back(F.bufC.p + (size_t)c0 * mm3);
      }
      fmm_upload(V.g_A, pa, st);
      fmm_upload(V.g_B, pb, st);
      fmm_upload(V.g_C, pc, st);
    }
  }
  size_t maxocc = 1;
  for (int l = 0; l <= L; ++l) maxocc = std::max(maxocc, (size_t)F.lev[l].nocc);
  F.tmpA.alloc(m * maxocc);
  F.tmpB.alloc(m * maxocc);
  {
    const int m3 = 3 * F.ns, mu3 = m3 + 1;
    for (int l = 2; l < L; ++l) {
      FmmLevel& P = F.lev[l];
      P.mm_m.clear(); P.mm_n.clear(); P.mm_k.clear(); P.mm_lda.clear(); P.mm_ldb.clear(); P.mm_ldc.clear();
      P.ll_k.clear(); P.ll_ldb.clear(); P.mm_alpha.clear();
      std::vector<const double*> ma, mb, la, lb;
      std::vector<double*> mc;
      for (int o = 0; o < 8; ++o) {
        const int c0 = P.oct_start[o], cnt = P.oct_start[o + 1] - c0;
        if (!cnt) continue;
        P.mm_m.push_back(m3); P.mm_n.push_back(cnt); P.mm_k.push_back(mu3); P.ll_k.push_back(m3);
        P.mm_lda.push_back(m3); P.mm_ldb.push_back(mu3); P.ll_ldb.push_back(m3); P.mm_ldc.push_back(m3);
        P.mm_alpha.push_back(1.0 / P.r);
        ma.push_back(F.M2M.p + (size_t)o * m3 * mu3);
        la.push_back(F.L2L.p + (size_t)o * m3 * m3);
        mb.push_back(F.tmpA.p + (size_t)c0 * mu3);
        lb.push_back(F.tmpA.p + (size_t)c0 * m3);
        mc.push_back(F.tmpB.p + (size_t)c0 * m3);
      }
      fmm_upload(P.mm_A, ma, st);
      fmm_upload(P.mm_B, mb, st);
      fmm_upload(P.ll_A, la, st);
      fmm_upload(P.ll_B, lb, st);
      fmm_upload(P.mm_C, mc, st);
    }
  }
  BPQN_CUDA(cudaStreamSynchronize(st));
}

static bool fmm_grouped() {
  static const bool grouped = !(getenv("BPQN_FMM_GROUPED") && getenv("BPQN_FMM_GROUPED")[0] == '0');
  return grouped;
}

// ------------------------------------------------------------------ apply
// out[N][3] = the K1 coarse sum (S and / or D) by the FMM, original node order.
void fmm_apply(Geom& g, const double* sigS, const double* sigD, double* out, cudaStream_t st) {
  Fmm& F = *g.fmm;
  const int N = g.n, L = F.L, ns = F.ns, m = 3 * ns, mu = m + 1;
  const size_t mm = (size_t)m * m, mmu = (size_t)m * mu;
  const bool doS = sigS != nullptr, doD = sigD != nullptr;
  const double cS = 1.0 / (8.0 * 3.14159265358979323846 * g.mu), cD = -3.0 / (4.0 * 3.14159265358979323846);
  k_fmm_records<<<(N + 255) / 256, 256, 0, st>>>(N, F.perm.p, g.src.p, sigS, sigD, cS, cD, F.rec.p);
  BPQN_CHECK_LAUNCH();
  FmmLevel& LV = F.lev[L];
  const double rad = FMM_OUT * LV.r;
  const int md = (doS && doD) ? MODE_SD : (doS ? MODE_S : MODE_D);
  // small leaves: the near-field items need only the records, so they start now on the caller's stream and the
  // tree pass runs beside them on a high-priority stream (its small GEMMs / gathers leave the FP64 pipe half
  // idle); the L2P items follow the tree pass, the per-target sum joins both (BPQN_FMM_OVERLAP=0: in order)
  static const bool use_seg = !(getenv("BPQN_FMM_SEG") && atoi(getenv("BPQN_FMM_SEG")) == 0);
  static const bool overlap = !(getenv("BPQN_FMM_OVERLAP") && getenv("BPQN_FMM_OVERLAP")[0] == '0');
  const bool seg = F.n_items > 0 && use_seg && !getenv("BPQN_FMM_LEAF_R");
  const cudaStream_t st_main = st;
  // forked apply: unused dynamic shared memory (PAD KB per CTA) caps the items' residency, so that the tree
  // pass's GEMM CTAs find registers beside them
  static const int pad_kb = getenv("BPQN_FMM_LEAF_PAD_KB") ? atoi(getenv("BPQN_FMM_LEAF_PAD_KB")) : 0;
  const size_t pad = (seg && overlap) ? (size_t)pad_kb * 1024 : 0;
  auto launch_items = [&](cudaStream_t ss, int i0, int cnt) {
    if (cnt <= 0) return;
    const int4* it = reinterpret_cast<const int4*>(F.leaf_items.p) + i0;
    // inner loop unrolled by 2 (measured: 1 -> 2.60, 2 -> 2.55, 4 -> 2.55 ms per c4 order-6 D apply)
    if (md == MODE_SD)
      k_fmm_leaf_seg<MODE_SD, 2><<<cnt, FL_T, pad, ss>>>(it, F.rec.p, F.leaf_start.p, F.leaf_nbr.p, F.surf.p, ns,
                                                       LV.ctr.p, rad, LV.deq.p, N, F.part.p);
    else if (md == MODE_S)
      k_fmm_leaf_seg<MODE_S, 2><<<cnt, FL_T, pad, ss>>>(it, F.rec.p, F.leaf_start.p, F.leaf_nbr.p, F.surf.p, ns,
                                                      LV.ctr.p, rad, LV.deq.p, N, F.part.p);
    else
      k_fmm_leaf_seg<MODE_D, 2><<<cnt, FL_T, pad, ss>>>(it, F.rec.p, F.leaf_start.p, F.leaf_nbr.p, F.surf.p, ns,
                                                      LV.ctr.p, rad, LV.deq.p, N, F.part.p);
    BPQN_CHECK_LAUNCH();
  };
  const bool forked = seg && overlap;
  // BPQN_FMM_TIMING=1 (development): event times of the two branches of a forked apply, printed after a sync
  static const bool dbg_t = getenv("BPQN_FMM_TIMING") != nullptr;
  static cudaEvent_t dbg_ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  if (dbg_t && !dbg_ev[0])
    for (auto& e : dbg_ev) BPQN_CUDA(cudaEventCreate(&e));
  if (forked) {
    if (!F.tree_stream) {
      int lo_pr = 0, hi_pr = 0;
      BPQN_CUDA(cudaDeviceGetStreamPriorityRange(&lo_pr, &hi_pr));
      BPQN_CUDA(cudaStreamCreateWithPriority(&F.tree_stream, cudaStreamNonBlocking, hi_pr));
      BPQN_CUDA(cudaEventCreateWithFlags(&F.ev_fork, cudaEventDisableTiming));
      BPQN_CUDA(cudaEventCreateWithFlags(&F.ev_join, cudaEventDisableTiming));
    }
    BPQN_CUDA(cudaEventRecord(F.ev_fork, st_main));
    BPQN_CUDA(cudaStreamWaitEvent(F.tree_stream, F.ev_fork, 0));
    if (dbg_t) BPQN_CUDA(cudaEventRecord(dbg_ev[0], st_main));
    launch_items(st_main, 0, F.n_near);
    if (dbg_t) BPQN_CUDA(cudaEventRecord(dbg_ev[1], st_main));
    st = F.tree_stream;  // the tree pass below
    if (dbg_t) BPQN_CUDA(cudaEventRecord(dbg_ev[2], st));
  }
  // upward: P2M at the leaves, check -> equivalent
  k_fmm_p2m<<<LV.nocc, 128, 0, st>>>(F.rec.p, F.leaf_start.p, F.surf.p, ns, LV.ctr.p, FMM_OUT * LV.r, doS, doD,
                                     LV.uck.p);
  BPQN_CHECK_LAUNCH();
  blas_dgemm(st, FMM_OP_N, FMM_OP_N, mu, LV.nocc, m, LV.r, F.UC2E.p, mu, LV.uck.p, m, 0.0, LV.ueq.p, mu);
  for (int l = L - 1; l >= 2; --l) {  // M2M: children (l + 1) -> parents (l), octant by octant
    FmmLevel& P = F.lev[l];
    FmmLevel& C = F.lev[l + 1];
    BPQN_CUDA(cudaMemsetAsync(P.uck.p, 0, 8 * (size_t)m * P.nocc, st));
    // all children octant-major in one gather, the 8 octant GEMMs as one grouped call, then each parent adds
    // its children's columns in octant order
    k_fmm_gather<<<fgrid((size_t)mu * P.n_child), 256, 0, st>>>(C.ueq.p, mu, P.ch_all.p, P.n_child, F.tmpA.p);
    BPQN_CHECK_LAUNCH();
    {
      const int G = (int)P.mm_m.size();
      if (!(fmm_grouped() && G > 0 &&
            blas_dgemm_grouped(st, G, P.mm_m.data(), P.mm_n.data(), P.mm_k.data(), P.mm_alpha.data(), P.mm_A.p,
                               P.mm_lda.data(), P.mm_B.p, P.mm_ldb.data(), P.mm_C.p, P.mm_ldc.data())))
        for (int o = 0; o < 8; ++o) {
          const int c0 = P.oct_start[o], cnt = P.oct_start[o + 1] - c0;
          if (!cnt) continue;
          blas_dgemm(st, FMM_OP_N, FMM_OP_N, m, cnt, mu, 1.0 / P.r, F.M2M.p + o * mmu, m,
                     F.tmpA.p + (size_t)c0 * mu, mu, 0.0, F.tmpB.p + (size_t)c0 * m, m);
        }
    }
    k_fmm_m2l_reduce<<<fgrid((size_t)m * P.nocc), 256, 0, st>>>(P.uck.p, m, P.nocc, P.par_ptr.p, P.par_pos.p,
                                                                F.tmpB.p);
    BPQN_CHECK_LAUNCH();
    blas_dgemm(st, FMM_OP_N, FMM_OP_N, mu, P.nocc, m, P.r, F.UC2E.p, mu, P.uck.p, m, 0.0, P.ueq.p, mu);
  }
  // downward: L2L from the parent, then M2L, then check -> equivalent
  for (int l = 2; l <= L; ++l) {
    FmmLevel& V = F.lev[l];
    BPQN_CUDA(cudaMemsetAsync(V.dck.p, 0, 8 * (size_t)m * V.nocc, st));
    if (l > 2) {
      FmmLevel& P = F.lev[l - 1];
      k_fmm_gather<<<fgrid((size_t)m * P.n_child), 256, 0, st>>>(P.deq.p, m, P.par_all.p, P.n_child, F.tmpA.p);
      BPQN_CHECK_LAUNCH();
      const int G = (int)P.mm_m.size();
      if (!(fmm_grouped() && G > 0 &&
            blas_dgemm_grouped(st, G, P.mm_m.data(), P.mm_n.data(), P.ll_k.data(), P.mm_alpha.data(), P.ll_A.p,
                               P.mm_lda.data(), P.ll_B.p, P.ll_ldb.data(), P.mm_C.p, P.mm_ldc.data())))
        for (int o = 0; o < 8; ++o) {
          const int c0 = P.oct_start[o], cnt = P.oct_start[o + 1] - c0;
          if (!cnt) continue;
          blas_dgemm(st, FMM_OP_N, FMM_OP_N, m, cnt, m, 1.0 / P.r, F.L2L.p + o * mm, m,
                     F.tmpA.p + (size_t)c0 * m, m, 0.0, F.tmpB.p + (size_t)c0 * m, m);
        }
      // every child has one parent: one scatter over all octants (d_ck was zeroed above)
      k_fmm_scatter_add<<<fgrid((size_t)m * P.n_child), 256, 0, st>>>(V.dck.p, m, P.ch_all.p, P.n_child, F.tmpB.p);
      BPQN_CHECK_LAUNCH();
    }
    if (V.n_pairs > 0 && F.m2l_comp) {
      // u~ = WV^T u_eq, per pair the rU x rV core, d_ck += WU (sum over the target's pairs)
      const int rU = F.rU, rV = F.rV;
      blas_dgemm(st, FMM_OP_T, FMM_OP_N, rV, V.nocc, mu, 1.0, F.WV.p, mu, V.ueq.p, mu, 0.0, F.tmpA.p, rV);
      k_fmm_gather<<<fgrid((size_t)rV * V.n_pairs), 256, 0, st>>>(F.tmpA.p, rV, V.m2l_src.p, V.n_pairs, F.bufB.p);
      BPQN_CHECK_LAUNCH();
      static const bool grouped = !(getenv("BPQN_FMM_GROUPED") && getenv("BPQN_FMM_GROUPED")[0] == '0');
      const int G = (int)V.g_m.size();
      if (!(grouped && G > 0 &&
            blas_dgemm_grouped(st, G, V.g_m.data(), V.g_n.data(), V.g_k.data(), V.g_alpha.data(), V.g_A.p,
                               V.g_lda.data(), V.g_B.p, V.g_ldb.data(), V.g_C.p, V.g_ldc.data())))
        for (int o = 0; o < FMM_NOFF; ++o) {
          const int c0 = V.off_start[o], cnt = V.off_start[o + 1] - c0;
          if (!cnt) continue;
          blas_dgemm(st, FMM_OP_N, FMM_OP_N, rU, cnt, rV, 1.0 / V.r, F.M2Lc.p + (size_t)o * rU * rV, rU,
                     F.bufB.p + (size_t)c0 * rV, rV, 0.0, F.bufC.p + (size_t)c0 * rU, rU);
        }
      BPQN_CUDA(cudaMemsetAsync(F.tmpB.p, 0, 8 * (size_t)rU * V.nocc, st));
      k_fmm_m2l_reduce<<<fgrid((size_t)rU * V.nocc), 256, 0, st>>>(F.tmpB.p, rU, V.nocc, V.tgt_ptr.p, V.tgt_pos.p,
                                                                   F.bufC.p);
      BPQN_CHECK_LAUNCH();
      blas_dgemm(st, FMM_OP_N, FMM_OP_N, m, V.nocc, rU, 1.0, F.WU.p, m, F.tmpB.p, rU, 1.0, V.dck.p, m);
    } else if (V.n_pairs > 0) {
      k_fmm_gather<<<fgrid((size_t)mu * V.n_pairs), 256, 0, st>>>(V.ueq.p, mu, V.m2l_src.p, V.n_pairs, F.bufB.p);
      BPQN_CHECK_LAUNCH();
      static const bool grouped = !(getenv("BPQN_FMM_GROUPED") && getenv("BPQN_FMM_GROUPED")[0] == '0');
      const int G = (int)V.g_m.size();
      if (!(grouped && G > 0 &&
            blas_dgemm_grouped(st, G, V.g_m.data(), V.g_n.data(), V.g_k.data(), V.g_alpha.data(), V.g_A.p,
                               V.g_lda.data(), V.g_B.p, V.g_ldb.data(), V.g_C.p, V.g_ldc.data())))
        for (int o = 0; o < FMM_NOFF; ++o) {
          const int c0 = V.off_start[o], cnt = V.off_start[o + 1] - c0;
          if (!cnt) continue;
          blas_dgemm(st, FMM_OP_N, FMM_OP_N, m, cnt, mu, 1.0 / V.r, F.M2L.p + o * mmu, m,
                     F.bufB.p + (size_t)c0 * mu, mu, 0.0, F.bufC.p + (size_t)c0 * m, m);
        }
      k_fmm_m2l_reduce<<<fgrid((size_t)m * V.nocc), 256, 0, st>>>(V.dck.p, m, V.nocc, V.tgt_ptr.p, V.tgt_pos.p,
                                                                  F.bufC.p);
      BPQN_CHECK_LAUNCH();
    }
    blas_dgemm(st, FMM_OP_N, FMM_OP_N, m, V.nocc, m, V.r, F.DC2E.p, m, V.dck.p, m, 0.0, V.deq.p, m);
  }
  // leaves: near field + L2P
  const int maxpts = g.fmm_max_leaf;  // the largest leaf sets the grid's second dimension
  // targets per thread: 3 share every staged source (large leaves, N = 589 824 at order 10: 43.7 ms); small
  // leaves (low orders, deeper trees) need the CTAs -- c4 at order 6: one target per thread 4.31 ms per D
  // apply, two 4.62, three 4.78 (profiles/r02_fmm_refine.md)
  int R = maxpts >= 3 * FL_T * 4 ? 3 : 1;
  if (const char* e = getenv("BPQN_FMM_LEAF_R")) R = std::max(1, std::min(3, atoi(e)));
  const dim3 lg(LV.nocc, (maxpts + FL_T * R - 1) / (FL_T * R));
  auto launch = [&](auto kern) {
    kern<<<lg, FL_T, 0, st>>>(F.rec.p, F.leaf_start.p, F.leaf_nbr.p, F.perm.p, F.surf.p, ns, LV.ctr.p, rad,
                              LV.deq.p, out);
  };
  if (seg) {
    if (forked) {  // L2P behind the tree pass, then join the caller's stream
      if (dbg_t) BPQN_CUDA(cudaEventRecord(dbg_ev[3], st));
      launch_items(st, F.n_near, F.n_items - F.n_near);
      if (dbg_t) BPQN_CUDA(cudaEventRecord(dbg_ev[4], st));
      BPQN_CUDA(cudaEventRecord(F.ev_join, st));
      BPQN_CUDA(cudaStreamWaitEvent(st_main, F.ev_join, 0));
    } else {
      launch_items(st, 0, F.n_items);
    }
    k_fmm_leaf_sum<<<(N + 255) / 256, 256, 0, st_main>>>(N, F.tparts.p, F.perm.p, F.part.p, out);
    BPQN_CHECK_LAUNCH();
    g.prof.launches += 10;
    if (dbg_t && forked) {
      BPQN_CUDA(cudaStreamSynchronize(st_main));
      float near_ms = 0, tree_ms = 0, l2p_ms = 0, tree_end = 0;
      cudaEventElapsedTime(&near_ms, dbg_ev[0], dbg_ev[1]);
      cudaEventElapsedTime(&tree_ms, dbg_ev[2], dbg_ev[3]);
      cudaEventElapsedTime(&l2p_ms, dbg_ev[3], dbg_ev[4]);
      cudaEventElapsedTime(&tree_end, dbg_ev[0], dbg_ev[4]);
      fprintf(stderr, "[bpqn fmm] near items %.3f ms | tree pass %.3f ms, L2P items %.3f ms (done %.3f ms after the fork)\n",
              near_ms, tree_ms, l2p_ms, tree_end);
    }
    return;
  }
  if (md == MODE_SD) {
    if (R == 3) launch(k_fmm_leaf<MODE_SD, 3>);
    else if (R == 2) launch(k_fmm_leaf<MODE_SD, 2>);
    else launch(k_fmm_leaf<MODE_SD, 1>);
  } else if (md == MODE_S) {
    if (R == 3) launch(k_fmm_leaf<MODE_S, 3>);
    else if (R == 2) launch(k_fmm_leaf<MODE_S, 2>);
    else launch(k_fmm_leaf<MODE_S, 1>);
  } else {
    if (R == 3) launch(k_fmm_leaf<MODE_D, 3>);
    else if (R == 2) launch(k_fmm_leaf<MODE_D, 2>);
    else launch(k_fmm_leaf<MODE_D, 1>);
  }
  BPQN_CHECK_LAUNCH();
  g.prof.launches += 8;
}

}  // namespace bpqn
