// The discrete layer operator on B200:
//   K1  all-pairs coarse-rule Stokeslet / stresslet summation (FP64 pipe bound),
//   K2  near-incidence correction: per (target, sphere) refined tensors in SH space [6][nb'] (HBM bound),
//   K3  per-sphere self operator Y = E X on FP64 tensor cores (mma.sync f64, DMMA),
//       whose epilogue also adds the K1 and K2 results.
// Operator definition O6 of DESIGN.md (paper: P:130-136, P:423-426 treat it as a
// black box).  Kernels written for sm_100a; no tcgen05 kind supports f64, so K3
// uses the DMMA path (measured 37.2 TFLOP/s on B200, same as DFMA).
#include <algorithm>
#include <atomic>

#include "bpqn_internal.h"

namespace bpqn {

// ------------------------------------------------------------------ K2
// Near-incidence correction, per incidence (target x_i, source sphere m):
//   u_i += sum_c sum_b T[sym(a,c)][b] coef_m[b][c]          refined rule (R8), SH space
//        - sum_{j in m} w_j K(x_i, y_j) sigma_j               the coarse pairs K1 added
// coef_m = analysis sigma_m (the Pi_p projection's SH coefficients, R7).  Blocks take
// chunks of incidences of one source sphere (K2 order, bpqn_internal.h), stage that
// sphere's nodes, weighted densities and coefficients in shared memory, and stream the
// [6][nb] tensors from HBM once per application (16-byte streaming loads); the coarse
// subtraction is recomputed from the staged nodes (~30 flops per pair, FP64 pipe).
// One incidence per half-warp; each stores its 3 values per incidence (k_row_reduce adds them per
// target row in a fixed order).

// coef[m][b][c] = sum_j A[b][j] sigma[m][j][c] (A row-major [nb][nq]); rows b in [nb, nbp) are zero.
// A small tiled GEMM: block = 32 rows of A x 8 spheres; its 256 threads form 4 groups that take
// interleaved slabs of 16 nodes (each thread 4 rows x 1 sphere x 3 components), then add their
// partial sums through shared memory; the KC_Z blocks along gridDim.z split the nodes and write
// one coefficient slab each (k2_near adds the slabs in a fixed order -- no atomics).  A is read
// once per 8 spheres (L2 traffic nb nq Np bytes).
constexpr int KC_BM = 32, KC_BS = 8, KC_JT = 16, KC_G = 4, KC_Z = 4;
__global__ void __launch_bounds__(256) k2_coef(int nq, int nb, int nbp, int np, const double* __restrict__ A,
                                               const double* __restrict__ sig, double* __restrict__ coef) {
  constexpr int NA = KC_G * KC_BM * (KC_JT + 1), NS = KC_G * KC_BS * KC_JT * 3;
  static_assert(NA + NS >= KC_G * 64 * 12, "reduction buffer");
  __shared__ double sm[NA + NS];
  double (*As)[KC_BM][KC_JT + 1] = reinterpret_cast<double (*)[KC_BM][KC_JT + 1]>(sm);
  double (*Ss)[KC_BS][KC_JT * 3] = reinterpret_cast<double (*)[KC_BS][KC_JT * 3]>(sm + NA);
  const int b0 = blockIdx.x * KC_BM, s0 = blockIdx.y * KC_BS;
  const int tid = threadIdx.x, grp = tid >> 6, t = tid & 63, tr = t & 7, ts = t >> 3;
  double c[4][3];
#pragma unroll
  for (int u = 0; u < 4; ++u) c[u][0] = c[u][1] = c[u][2] = 0.0;
  const int jlen = (nq + gridDim.z - 1) / gridDim.z;  // this block's node range [ja, je)
  const int ja = blockIdx.z * jlen, je = min(nq, ja + jlen);
  for (int jr = ja; jr < je; jr += KC_G * KC_JT) {
    // every thread helps stage all KC_G slabs of this round
    for (int e = tid; e < KC_G * KC_BM * KC_JT; e += 256) {
      const int g = e / (KC_BM * KC_JT), rem = e - g * (KC_BM * KC_JT), r = rem / KC_JT, jj = rem - r * KC_JT;
      const int j = jr + g * KC_JT + jj;
      As[g][r][jj] = (b0 + r < nb && j < je) ? A[(size_t)(b0 + r) * nq + j] : 0.0;
    }
    for (int e = tid; e < KC_G * KC_BS * KC_JT * 3; e += 256) {
      const int g = e / (KC_BS * KC_JT * 3), rem = e - g * (KC_BS * KC_JT * 3), sp = rem / (KC_JT * 3),
                k = rem - sp * (KC_JT * 3);
      const int j = jr + g * KC_JT + k / 3;
      Ss[g][sp][k] = (s0 + sp < np && j < je) ? sig[((size_t)(s0 + sp) * nq + jr + g * KC_JT) * 3 + k] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int jj = 0; jj < KC_JT; ++jj) {
      const double q0 = Ss[grp][ts][3 * jj], q1 = Ss[grp][ts][3 * jj + 1], q2 = Ss[grp][ts][3 * jj + 2];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double av = As[grp][4 * tr + u][jj];
        c[u][0] = fma(av, q0, c[u][0]);
        c[u][1] = fma(av, q1, c[u][1]);
        c[u][2] = fma(av, q2, c[u][2]);
      }
    }
    __syncthreads();
  }
  // reduce the KC_G groups' partial sums (the staging buffer reused as [KC_G][64 threads][12])
  double* red = sm;
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int k = 0; k < 3; ++k) red[(grp * 64 + t) * 12 + 3 * u + k] = c[u][k];
  __syncthreads();
  if (grp != 0 || s0 + ts >= np) return;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int bb = b0 + 4 * tr + u;
    if (bb >= nbp) continue;
    double* o = coef + (size_t)blockIdx.z * np * nbp * 3 + ((size_t)(s0 + ts) * nbp + bb) * 3;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      double v = 0.0;
#pragma unroll
      for (int g = 0; g < KC_G; ++g) v += red[(g * 64 + t) * 12 + 3 * u + k];
      o[k] = v;  // this node slab's coefficient
    }
  }
}

struct K2Params {
  const int *chunks, *cm_t, *cm_m;
  const double *X, *src;         // node positions [N][3]; records {y, w, n, 0} [N][8]
  const double* centers;         // [np][3]
  double a;
  const double *TS, *TD;         // [n_inc][6][nbp] or null (nbp = nb rounded up to even)
  const double *coefS, *coefD;   // [KC_Z][np][nbp][3] node-slab partial coefficients
  const double *sigS, *sigD;     // [N][3]
  int np, nq, nbp, t0, t1;       // targets outside [t0, t1) are skipped (sharding)
  double cS, cD;                 // 1/(8 pi mu), -3/(4 pi)
  double* pinc;                  // [n_inc][3] per-incidence sums (K2 order), summed per row by k_row_reduce
};

// u[a] += sum_c T[sym(a,c)] c[c] over the packed symmetric rows, streamed in b pairs
__device__ __forceinline__ void k2_refined(const double* __restrict__ T, const double* __restrict__ cf, int nbp,
                                           int hl, double& u0, double& u1, double& u2) {
  const double2* T2 = reinterpret_cast<const double2*>(T);
  const int nb2 = nbp >> 1;
#pragma unroll 2
  for (int b2 = hl; b2 < nb2; b2 += 16) {
    double2 t[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) t[q] = __ldcs(T2 + q * nb2 + b2);
    const double* c = cf + 6 * b2;  // coefficients of b = 2 b2 and 2 b2 + 1
    u0 = fma(t[0].x, c[0], fma(t[1].x, c[1], fma(t[2].x, c[2], u0)));
    u1 = fma(t[1].x, c[0], fma(t[3].x, c[1], fma(t[4].x, c[2], u1)));
    u2 = fma(t[2].x, c[0], fma(t[4].x, c[1], fma(t[5].x, c[2], u2)));
    u0 = fma(t[0].y, c[3], fma(t[1].y, c[4], fma(t[2].y, c[5], u0)));
    u1 = fma(t[1].y, c[3], fma(t[3].y, c[4], fma(t[4].y, c[5], u1)));
    u2 = fma(t[2].y, c[3], fma(t[4].y, c[4], fma(t[5].y, c[5], u2)));
  }
}

__global__ void __launch_bounds__(256, 4) k2_near(K2Params P) {
  extern __shared__ __align__(16) double k2s[];
  const int nq = P.nq, nb = P.nbp;
  const bool doS = P.TS != nullptr, doD = P.TD != nullptr;
  double* sy = k2s;                            // [nq][3] node positions
  double* sqD = sy + 3 * nq;                   // [nq][3] cD w sigmaD
  double* sqS = sqD + (doD ? 3 * nq : 0);      // [nq][3] cS w sigmaS
  double* scD = sqS + (doS ? 3 * nq : 0);      // [nb][3]
  double* scS = scD + (doD ? 3 * nb : 0);      // [nb][3]
  const int beg = P.chunks[2 * blockIdx.x], end = P.chunks[2 * blockIdx.x + 1];
  const int m = P.cm_m[beg];
  const size_t j0 = (size_t)m * nq;
  for (int e = threadIdx.x; e < 3 * nq; e += blockDim.x) {
    const double w = P.src[8 * (j0 + e / 3) + 3];
    sy[e] = P.X[3 * j0 + e];
    if (doD) sqD[e] = P.cD * w * P.sigD[3 * j0 + e];
    if (doS) sqS[e] = P.cS * w * P.sigS[3 * j0 + e];
  }
  const size_t slab = (size_t)P.np * nb * 3;
  for (int e = threadIdx.x; e < 3 * nb; e += blockDim.x) {
    double cd = 0.0, cs = 0.0;
#pragma unroll
    for (int z = 0; z < KC_Z; ++z) {  // node slabs in a fixed order
      if (doD) cd += P.coefD[z * slab + (size_t)m * nb * 3 + e];
      if (doS) cs += P.coefS[z * slab + (size_t)m * nb * 3 + e];
    }
    if (doD) scD[e] = cd;
    if (doS) scS[e] = cs;
  }
  const double cm0 = P.centers[3 * m], cm1 = P.centers[3 * m + 1], cm2 = P.centers[3 * m + 2];
  const double inv2a = 0.5 / P.a, a2 = P.a * P.a;
  __syncthreads();
  // one incidence per half-warp (two latency chains per warp, better lane use at small p)
  const int lane = threadIdx.x & 31, hl = lane & 15, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const unsigned hmask = 0xffffu << (lane & 16);
  for (int pos = beg + 2 * warp + (lane >> 4); pos < end; pos += 2 * nw) {
    const int i = P.cm_t[pos];
    if (i < P.t0 || i >= P.t1) continue;
    const double x0 = P.X[3 * (size_t)i], x1 = P.X[3 * (size_t)i + 1], x2 = P.X[3 * (size_t)i + 2];
    double u0 = 0.0, u1 = 0.0, u2 = 0.0;
    if (doD) k2_refined(P.TD + (size_t)pos * 6 * nb, scD, nb, hl, u0, u1, u2);
    if (doS) k2_refined(P.TS + (size_t)pos * 6 * nb, scS, nb, hl, u0, u1, u2);
    // minus the coarse pairs: K_D q = cD w (r.n)(r.q) r / rho^5, G f = cS w (f / rho + (r.f) r / rho^3);
    // on sphere m, r.n_y = h - rho^2 / (2a) with h = (|x - c_m|^2 - a^2) / (2a)
    const double d0 = x0 - cm0, d1 = x1 - cm1, d2 = x2 - cm2;
    const double h = (fma(d2, d2, fma(d1, d1, d0 * d0)) - a2) * inv2a;
#pragma unroll 4
    for (int j = hl; j < nq; j += 16) {
      const double r0 = x0 - sy[3 * j], r1 = x1 - sy[3 * j + 1], r2 = x2 - sy[3 * j + 2];
      const double rr = fma(r2, r2, fma(r1, r1, r0 * r0));
      double ir;  // rr^-1/2: MUFU.RSQ64H seed + (1-e)^-1/2 series to e^2 (|e| <= 2^-19, as K1)
      asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(ir) : "d"(rr));
      {
        const double e = fma(-rr, ir * ir, 1.0);
        ir = fma(ir * e, fma(e, 0.375, 0.5), ir);
      }
      const double ir2 = ir * ir, ir3 = ir * ir2;
      double t = 0.0;
      if (doD) {
        const double rn = fma(rr, -inv2a, h);
        const double rq = fma(r2, sqD[3 * j + 2], fma(r1, sqD[3 * j + 1], r0 * sqD[3 * j]));
        t = (rn * rq) * (ir3 * ir2);
      }
      if (doS) {
        const double rf = fma(r2, sqS[3 * j + 2], fma(r1, sqS[3 * j + 1], r0 * sqS[3 * j]));
        t = fma(rf, ir3, t);
        u0 = fma(-sqS[3 * j], ir, u0);
        u1 = fma(-sqS[3 * j + 1], ir, u1);
        u2 = fma(-sqS[3 * j + 2], ir, u2);
      }
      u0 = fma(-t, r0, u0);
      u1 = fma(-t, r1, u1);
      u2 = fma(-t, r2, u2);
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) {
      u0 += __shfl_xor_sync(hmask, u0, o);
      u1 += __shfl_xor_sync(hmask, u1, o);
      u2 += __shfl_xor_sync(hmask, u2, o);
    }
    if (hl == 0) {
      P.pinc[3 * (size_t)pos] = u0;
      P.pinc[3 * (size_t)pos + 1] = u1;
      P.pinc[3 * (size_t)pos + 2] = u2;
    }
  }
}

// K2 into the per-incidence partials g.k2_pinc (summed per target row by k_row_reduce).
void launch_near(Geom& g, const double* sigS, const double* sigD, cudaStream_t st) {
  if (g.n_inc == 0) return;
  const bool doS = sigS && g.T_S.p, doD = sigD != nullptr;
  if (!doS && !doD) return;
  const int nq = g.nq, nb = g.nb;
  const int nbp = (nb + 1) & ~1;
  BPQN_REQUIRE(g.coef.n >= (size_t)2 * KC_Z * g.np * nbp * 3, "K2 workspace too small (layer_reserve)");
  double* coefD = g.coef.p;
  double* coefS = g.coef.p + (size_t)KC_Z * g.np * nbp * 3;
  // node ranges split over KC_Z blocks for parallelism, one coefficient slab each
  const dim3 cgrid((nbp + KC_BM - 1) / KC_BM, (g.np + KC_BS - 1) / KC_BS, KC_Z);
  if (doD) {
    k2_coef<<<cgrid, 256, 0, st>>>(nq, nb, nbp, g.np, g.analysis.p, sigD, coefD);
    BPQN_CHECK_LAUNCH();
    g.prof.launches++;
  }
  if (doS) {
    k2_coef<<<cgrid, 256, 0, st>>>(nq, nb, nbp, g.np, g.analysis.p, sigS, coefS);
    BPQN_CHECK_LAUNCH();
    g.prof.launches++;
  }
  K2Params P{};
  P.chunks = g.chunks.p;
  P.cm_t = g.cm_t.p;
  P.cm_m = g.cm_m.p;
  P.X = g.X.p;
  P.src = g.src.p;
  P.centers = g.centers_d.p;
  P.a = g.a;
  P.TS = doS ? g.T_S.p : nullptr;
  P.TD = doD ? g.T_D.p : nullptr;
  P.coefS = coefS;
  P.coefD = coefD;
  P.sigS = sigS;
  P.sigD = sigD;
  P.np = g.np;
  P.nq = nq;
  P.nbp = nbp;
  P.t0 = g.sharded() ? g.sh_t0 : 0;
  P.t1 = g.sharded() ? g.sh_t1 : g.n;
  P.cS = 1.0 / (8.0 * 3.14159265358979323846 * g.mu);
  P.cD = -3.0 / (4.0 * 3.14159265358979323846);
  P.pinc = g.k2_pinc.p;
  const int smem = (3 * nq + (doD ? 3 * nq + 3 * nbp : 0) + (doS ? 3 * nq + 3 * nbp : 0)) * 8;
  static std::atomic<int> attr{48 * 1024};  // the opt-in limit only grows
  if (smem > attr.load()) {
    BPQN_CUDA(cudaFuncSetAttribute(k2_near, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr.store(smem);
  }
  k2_near<<<g.n_chunks, 256, smem, st>>>(P);
  BPQN_CHECK_LAUNCH();
  g.prof.launches++;
}

// ------------------------------------------------------------------ K3
// C[M x Np] (column n = sphere n, contiguous M = 3nq) = E[M x M] X[M x Np], E row-major,
// the same for every sphere (translation invariance of the self rule).  FP64 tensor
// cores via mma.sync m8n8k4 (DMMA; tcgen05 has no f64 kind).  CTA tile 64 x 72
// (8 warps, each one 8-row strip x 9 n8 tiles), K in stages of 16 through a 3-deep
// cp.async ring (zero-filled tails), split-K over gridDim.z with a fixed-order reduction of the
// partial tiles, accumulated into an output that k_row_reduce initialised with the K1 + K2 sums.
constexpr int K3_BM = 64, K3_BN = 72, K3_BK = 16, K3_ST = 3, K3_LDA = K3_BK + 4;  // LDA 20: conflict-free fragments
constexpr int K3_SMEM = K3_ST * (K3_BM + K3_BN) * K3_LDA * 8;

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const int sz = valid ? 16 : 0;  // 0 -> zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(sz) : "memory");
}

// Split-K without atomics: with gridDim.z > 1 every CTA stores its 64 x 72 partial tile in
// part[z][tile]; the last CTA of a tile to arrive (per-tile counter, reset by that CTA for the
// next launch or graph replay) adds the ks partials in z order to out -- a fixed summation
// order, so the result is bit-reproducible.  With one split the CTA writes out directly.
__global__ void __launch_bounds__(256) k3_self_gemm(int M, int Nn, int kchunk, const double* __restrict__ E,
                                                    const double* __restrict__ X, double* out, int accumulate,
                                                    double* __restrict__ part, unsigned* cnt) {
  extern __shared__ __align__(16) double k3_dyn[];
  __shared__ unsigned s_last;
  double (*As)[K3_BM][K3_LDA] = reinterpret_cast<double (*)[K3_BM][K3_LDA]>(k3_dyn);
  double (*Bs)[K3_BN][K3_LDA] = reinterpret_cast<double (*)[K3_BN][K3_LDA]>(k3_dyn + K3_ST * K3_BM * K3_LDA);
  const int m0 = blockIdx.x * K3_BM, n0 = blockIdx.y * K3_BN;
  const int kb = blockIdx.z * kchunk, ke = min(M, kb + kchunk);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;
  double acc[9][2];
#pragma unroll
  for (int j = 0; j < 9; ++j) acc[j][0] = acc[j][1] = 0.0;
  const int nst = (ke - kb + K3_BK - 1) / K3_BK;
  auto load = [&](int s, int k0) {
    // A: 64 rows x 16 doubles = 512 chunks of 16 B; B: 72 cols x 16 = 576 chunks
    for (int c = tid; c < K3_BM * (K3_BK / 2) + K3_BN * (K3_BK / 2); c += 256) {
      if (c < K3_BM * (K3_BK / 2)) {
        const int r = c >> 3, kk = (c & 7) * 2;
        const int gr = m0 + r, gk = k0 + kk;
        const bool v = gr < M && gk < ke;
        cp_async16(&As[s][r][kk], v ? E + (size_t)gr * M + gk : E, v);
      } else {
        const int c2 = c - K3_BM * (K3_BK / 2);
        const int nn = c2 >> 3, kk = (c2 & 7) * 2;
        const int gn = n0 + nn, gk = k0 + kk;
        const bool v = gn < Nn && gk < ke;
        cp_async16(&Bs[s][nn][kk], v ? X + (size_t)gn * M + gk : X, v);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
#pragma unroll
  for (int s = 0; s < K3_ST - 1; ++s) {
    if (s < nst) load(s, kb + s * K3_BK);
    else asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int st = 0; st < nst; ++st) {
    asm volatile("cp.async.wait_group %0;" ::"n"(K3_ST - 2) : "memory");
    __syncthreads();
    const int nxt = st + K3_ST - 1;
    if (nxt < nst) load(nxt % K3_ST, kb + nxt * K3_BK);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    const int s = st % K3_ST;
#pragma unroll
    for (int kk = 0; kk < K3_BK; kk += 4) {
      const double a = As[s][warp * 8 + g][kk + t4];
#pragma unroll
      for (int j = 0; j < 9; ++j) dmma884(acc[j][0], acc[j][1], a, Bs[s][j * 8 + g][kk + t4]);
    }
  }
  // epilogue: fragment row g, cols 2 t4 + {0, 1} of each n8 tile
  const int row = m0 + warp * 8 + g;
  const int ks = gridDim.z;
  if (ks > 1) {
    const size_t tile = (size_t)blockIdx.y * gridDim.x + blockIdx.x;
    const size_t ntile = (size_t)gridDim.x * gridDim.y;
    double* mine = part + ((size_t)blockIdx.z * ntile + tile) * (K3_BM * K3_BN);
#pragma unroll
    for (int j = 0; j < 9; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) mine[(warp * 8 + g) * K3_BN + j * 8 + 2 * t4 + h] = acc[j][h];
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(cnt + tile, 1u) == (unsigned)(ks - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
#pragma unroll
    for (int j = 0; j < 9; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double v = 0.0;
        for (int z = 0; z < ks; ++z)
          v += __ldcg(part + ((size_t)z * ntile + tile) * (K3_BM * K3_BN) + (warp * 8 + g) * K3_BN + j * 8 + 2 * t4 + h);
        acc[j][h] = v;
      }
    if (tid == 0) cnt[tile] = 0u;  // ready for the next launch / graph replay
  }
  if (row < M) {
#pragma unroll
    for (int j = 0; j < 9; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = n0 + j * 8 + 2 * t4 + h;
        if (col < Nn) {
          double* o = out + (size_t)col * M + row;
          *o = accumulate ? *o + acc[j][h] : acc[j][h];
        }
      }
  }
}

// split-K factor: about two waves of CTAs over the GPU, K chunks of >= 8 stages; one split
// (a single writer) when sharded
static int k3_splits(const Geom& g, int mt, int nt, int M) {
  int ks = std::max(1, std::min((2 * g.sms + mt * nt - 1) / (mt * nt), (M + 8 * K3_BK - 1) / (8 * K3_BK)));
  if (g.sharded()) ks = 1;
  int kchunk = (M + ks - 1) / ks;
  kchunk = ((kchunk + K3_BK - 1) / K3_BK) * K3_BK;
  return (M + kchunk - 1) / kchunk;
}

void launch_self_gemm(Geom& g, const double* E, const double* X, double* out, int accumulate, cudaStream_t st,
                      int s0, int s1) {
  // spheres [s0, s1) only (sharded operator); columns are contiguous per sphere
  if (s1 < 0) s1 = g.np;
  const int M = 3 * g.nq, ncol = s1 - s0;
  if (ncol <= 0) return;
  const size_t off = (size_t)M * s0;
  X += off;
  out += off;
  const int mt = (M + K3_BM - 1) / K3_BM, nt = (ncol + K3_BN - 1) / K3_BN;
  const int ks = k3_splits(g, mt, nt, M);
  const int kchunk = ((((M + ks - 1) / ks) + K3_BK - 1) / K3_BK) * K3_BK;
  BPQN_REQUIRE(ks == 1 || (g.k3_part.n >= (size_t)ks * mt * nt * K3_BM * K3_BN && g.k3_cnt.n >= (size_t)mt * nt),
               "K3 workspace too small (layer_reserve)");
  dim3 grid(mt, nt, ks);
  static bool attr = false;
  if (!attr) {
    BPQN_CUDA(cudaFuncSetAttribute(k3_self_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, K3_SMEM));
    attr = true;
  }
  k3_self_gemm<<<grid, 256, K3_SMEM, st>>>(M, ncol, kchunk, E, X, out, accumulate, g.k3_part.p, g.k3_cnt.p);
  BPQN_CHECK_LAUNCH();
  g.prof.launches += 1;
}

// K2 and K3 workspace, allocated at geometry init / update (no allocation in the hot calls).
void layer_reserve(Geom& g) {
  const int nbp = (g.nb + 1) & ~1;
  g.coef.ensure((size_t)2 * KC_Z * g.np * nbp * 3);
  g.k2_pinc.ensure(3 * (size_t)std::max<long long>(g.n_inc, 1));
  const int M = 3 * g.nq, mt = (M + K3_BM - 1) / K3_BM, nt = (g.np + K3_BN - 1) / K3_BN;
  const int ks = k3_splits(g, mt, nt, M);
  g.k3_part.ensure((size_t)std::max(ks, 1) * mt * nt * K3_BM * K3_BN);
  if (g.k3_cnt.n < (size_t)mt * nt) {
    g.k3_cnt.alloc((size_t)mt * nt);
    BPQN_CUDA(cudaMemset(g.k3_cnt.p, 0, sizeof(unsigned) * mt * nt));
  }
}

// Sharded operator (bpqn_geometry_shard): gather every rank's owned rows into `out`.
__global__ void k_shard_pack(const double* __restrict__ out, int t0, int nrow, double* __restrict__ send, int rows) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= 3 * rows) return;
  send[e] = e < 3 * nrow ? out[3 * (size_t)t0 + e] : 0.0;
}

__global__ void k_shard_unpack(const double* __restrict__ recv, int world, int rows, int np, int nq,
                               double* __restrict__ out) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= 3LL * rows * world) return;
  const int r = (int)(e / (3LL * rows)), k = (int)(e - 3LL * rows * r);
  const int s0 = (int)((long long)np * r / world), s1 = (int)((long long)np * (r + 1) / world);
  if (k < 3 * (s1 - s0) * nq) out[3 * (size_t)s0 * nq + k] = recv[e];
}

// reduce-scatter of the sharded symmetric K1's partial sums: send[r][k] = far rows of rank r
__global__ void k_rs_pack(const double* __restrict__ far, int world, int rows, int np, int nq,
                          double* __restrict__ send) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= 3LL * rows * world) return;
  const int r = (int)(e / (3LL * rows)), k = (int)(e - 3LL * rows * r);
  const int s0 = (int)((long long)np * r / world), s1 = (int)((long long)np * (r + 1) / world);
  send[e] = k < 3 * (s1 - s0) * nq ? far[3 * (size_t)s0 * nq + k] : 0.0;
}

// reduce-scatter of the sharded symmetric K1 partial sums into the owned rows of far: NCCL on the
// given stream (library communicator), or the caller's callback after a stream sync
static void shard_reduce_scatter(Geom& g, double* far, cudaStream_t st) {
  const long long tot = 3LL * g.sh_rows * g.shard_world;
  double* send = g.nccl_comm ? g.sh_own_rs_send.p : g.sh_rs_send;
  double* recv = g.nccl_comm ? g.sh_own_rs_recv.p : g.sh_rs_recv;
  k_rs_pack<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(far, g.shard_world, g.sh_rows, g.np, g.nq, send);
  BPQN_CHECK_LAUNCH();
  if (g.nccl_comm) {
    comm_reduce_scatter(g, send, recv, 3 * (size_t)g.sh_rows, st);
  } else {
    BPQN_CUDA(cudaStreamSynchronize(st));
    if (g.sh_rs_fn(g.sh_rs_user) != 0) throw Error{BPQN_ERR_CUDA, "shard reduce-scatter callback failed"};
  }
  // the owned rows of far <- the sum over ranks
  BPQN_CUDA(cudaMemcpyAsync(far + 3 * (size_t)g.sh_t0, recv, sizeof(double) * 3 * (size_t)(g.sh_t1 - g.sh_t0),
                            cudaMemcpyDeviceToDevice, st));
  g.prof.launches += 1;
}

static void shard_exchange(Geom& g, double* out, cudaStream_t st) {
  const int nrow = g.sh_t1 - g.sh_t0;
  double* send = g.nccl_comm ? g.sh_own_send.p : g.sh_send;
  double* recv = g.nccl_comm ? g.sh_own_recv.p : g.sh_recv;
  k_shard_pack<<<(3 * g.sh_rows + 255) / 256, 256, 0, st>>>(out, g.sh_t0, nrow, send, g.sh_rows);
  BPQN_CHECK_LAUNCH();
  if (g.nccl_comm) {
    comm_allgather(g, send, recv, 3 * (size_t)g.sh_rows, st);
  } else {
    BPQN_CUDA(cudaStreamSynchronize(st));
    if (g.sh_fn(g.sh_user) != 0) throw Error{BPQN_ERR_CUDA, "shard all-gather callback failed"};
  }
  const long long tot = 3LL * g.sh_rows * g.shard_world;
  k_shard_unpack<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(recv, g.shard_world, g.sh_rows, g.np, g.nq, out);
  BPQN_CHECK_LAUNCH();
  g.prof.launches += 2;
}

// ------------------------------------------------------------------ operator
// out = coarse all-pairs + near corrections + self blocks, for densities sigS
// (single layer, self matrix Es) and sigD (double layer, self matrix Ed).
void apply_operator(Geom& g, const double* sigS, const double* sigD, const double* Es, const double* Ed,
                    double* out, cudaStream_t st) {
  int mode = (sigS && sigD) ? MODE_SD : (sigS ? MODE_S : MODE_D);
  Profile& P = g.prof;
  // Optionally (BPQN_OVERLAP_K2=1) K2 (HBM bound) runs on a side stream concurrently
  // with K1 (FP64 bound).  Measured on B200 at c4: no gain -- K1 slows by K2's whole
  // duration -- so K2 runs in order by default.
  if (!g.side) {
    BPQN_CUDA(cudaStreamCreateWithFlags(&g.side, cudaStreamNonBlocking));
    BPQN_CUDA(cudaEventCreateWithFlags(&g.ev_fork, cudaEventDisableTiming));
    BPQN_CUDA(cudaEventCreateWithFlags(&g.ev_join, cudaEventDisableTiming));
  }
  bool overlap = g.overlap_k2;
  if (!overlap && g.fmm && g.fmm_on && g.fmm_max_leaf < 768) {  // (large leaves, N = 589 824: 2 % slower)
    // with the FMM far field the co-resident kernels are small (leaf items of 64 threads, GEMMs, gathers), so
    // the HBM-bound K2 does fit beside them: c4 order-6 refined MVP 321 -> 313 ms (BPQN_FMM_OVERLAP=0: in
    // order).  Not while the GMRES cycle is being captured (the captured step stays a single-stream chain).
    static const bool fmm_ov = !(getenv("BPQN_FMM_OVERLAP") && getenv("BPQN_FMM_OVERLAP")[0] == '0');
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (fmm_ov && cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone) overlap = true;
  }
  cudaStream_t sk2 = overlap ? g.side : st;
  cudaEvent_t* ev = nullptr;
  if (P.events) {
    while (P.pool.size() < P.used + 5) {
      cudaEvent_t e;
      BPQN_CUDA(cudaEventCreate(&e));
      P.pool.push_back(e);
    }
    ev = P.pool.data() + P.used;
    P.used += 5;
  }
  const bool sharded = g.sharded();
  const int s0 = sharded ? g.sh_s0 : 0, s1 = sharded ? g.sh_s1 : g.np;
  const int r0 = sharded ? g.sh_t0 : 0, r1 = sharded ? g.sh_t1 : g.n;
  if (sharded && g.nccl_comm && k1_sharded_symmetric(g)) {
    // K1 over this rank's units -> far (all rows); its NCCL reduce-scatter on the side stream
    // overlaps K2 on the main stream; then out = far(owned) + K2, K3, all-gather
    if (ev) BPQN_CUDA(cudaEventRecord(ev[0], st));
    launch_allpairs(g, mode, sigS, sigD, g.far.p, st);
    if (ev) {
      BPQN_CUDA(cudaEventRecord(ev[1], st));
      P.allpairs_flop += (double)g.n * ((double)g.n / g.shard_world) * allpairs_flops_per_pair(mode);
    }
    launch_row_reduce(g, true, nullptr, false, g.far.p, 0, g.n, st);
    BPQN_CUDA(cudaEventRecord(g.ev_fork, st));
    BPQN_CUDA(cudaStreamWaitEvent(g.side, g.ev_fork, 0));
    shard_reduce_scatter(g, g.far.p, g.side);
    BPQN_CUDA(cudaEventRecord(g.ev_join, g.side));
    if (ev) BPQN_CUDA(cudaEventRecord(ev[2], st));
    launch_near(g, sigS, sigD, st);
    if (ev) BPQN_CUDA(cudaEventRecord(ev[3], st));
    BPQN_CUDA(cudaStreamWaitEvent(st, g.ev_join, 0));
    launch_row_reduce(g, false, g.far.p, true, out, r0, r1, st);
    if (sigS) launch_self_gemm(g, Es, sigS, out, 1, st, s0, s1);
    if (sigD) launch_self_gemm(g, Ed, sigD, out, 1, st, s0, s1);
    shard_exchange(g, out, st);
    if (ev) BPQN_CUDA(cudaEventRecord(ev[4], st));
    return;
  }
  if (overlap) {
    BPQN_CUDA(cudaEventRecord(g.ev_fork, st));
    BPQN_CUDA(cudaStreamWaitEvent(g.side, g.ev_fork, 0));
  }
  if (ev) BPQN_CUDA(cudaEventRecord(ev[2], sk2));
  launch_near(g, sigS, sigD, sk2);
  if (ev) BPQN_CUDA(cudaEventRecord(ev[3], sk2));
  if (g.fmm && g.fmm_on) {  // far-field FMM in place of K1 (fmm.cu): the coarse sum into far, then far + K2, K3
    BPQN_REQUIRE(!sharded, "the FMM far field does not combine with sharding");
    if (ev) BPQN_CUDA(cudaEventRecord(ev[0], st));
    fmm_apply(g, sigS, sigD, g.far.p, st);
    if (ev) {
      BPQN_CUDA(cudaEventRecord(ev[1], st));
      P.allpairs_flop += (double)g.n * (double)g.n * allpairs_flops_per_pair(mode);  // nominal
    }
    if (overlap) {
      BPQN_CUDA(cudaEventRecord(g.ev_join, g.side));
      BPQN_CUDA(cudaStreamWaitEvent(st, g.ev_join, 0));
    }
    launch_row_reduce(g, false, g.far.p, true, out, r0, r1, st);
    if (sigS) launch_self_gemm(g, Es, sigS, out, 1, st, s0, s1);
    if (sigD) launch_self_gemm(g, Ed, sigD, out, 1, st, s0, s1);
    if (ev) BPQN_CUDA(cudaEventRecord(ev[4], st));
    return;
  }
  if (ev) BPQN_CUDA(cudaEventRecord(ev[0], st));
  launch_allpairs(g, mode, sigS, sigD, g.far.p, st);
  if (ev) {
    BPQN_CUDA(cudaEventRecord(ev[1], st));
    // this rank's share of the nominal N^2 pairs
    const double ntg = sharded ? (k1_sharded_symmetric(g) ? (double)g.n / g.shard_world
                                                          : (double)(g.sh_t1 - g.sh_t0))
                               : (double)g.n;
    P.allpairs_flop += (double)g.n * ntg * allpairs_flops_per_pair(mode);
  }
  if (overlap) {
    BPQN_CUDA(cudaEventRecord(g.ev_join, g.side));
    BPQN_CUDA(cudaStreamWaitEvent(st, g.ev_join, 0));
  }
  // out = K1 + K2 (fixed-order row sums), then the self blocks K3 accumulate into it
  if (sharded && k1_sharded_symmetric(g)) {
    launch_row_reduce(g, true, nullptr, false, g.far.p, 0, g.n, st);  // this rank's K1 partials, all rows
    shard_reduce_scatter(g, g.far.p, st);                              // owned rows of far = sum over ranks
    launch_row_reduce(g, false, g.far.p, true, out, r0, r1, st);
  } else {
    launch_row_reduce(g, true, nullptr, true, out, r0, r1, st);  // K1 segment partials (either kernel)
  }
  if (sigS) launch_self_gemm(g, Es, sigS, out, 1, st, s0, s1);
  if (sigD) launch_self_gemm(g, Ed, sigD, out, 1, st, s0, s1);
  if (sharded) shard_exchange(g, out, st);
  if (ev) BPQN_CUDA(cudaEventRecord(ev[4], st));
}

// Sum the recorded operator timings (one host sync) and recycle the events.
// Per application: [2]/[3] around K2 (side stream when overlapped), [0]/[1] around K1,
// [4] main after K3.  ms_self = [1] -> [4] (K3, plus any
// wait for an overlapped K2 that outlasted K1).
void profile_collect(Geom& g) {
  Profile& P = g.prof;
  if (P.used == 0) return;
  BPQN_CUDA(cudaEventSynchronize(P.pool[P.used - 1]));
  for (size_t k = 0; k < P.used; k += 5) {
    float a = 0, b = 0, c = 0;
    BPQN_CUDA(cudaEventElapsedTime(&a, P.pool[k], P.pool[k + 1]));
    BPQN_CUDA(cudaEventElapsedTime(&b, P.pool[k + 2], P.pool[k + 3]));
    BPQN_CUDA(cudaEventElapsedTime(&c, P.pool[k + 1], P.pool[k + 4]));
    P.ms_allpairs += a;
    P.ms_near += b;
    P.ms_self += c;
  }
  P.used = 0;
}

}  // namespace bpqn
