// The discrete layer operator on B200:
//   K1  all-pairs coarse-rule Stokeslet / stresslet summation (FP64 pipe bound),
//   K2  near-incidence correction: per (target, sphere) [3][3nq] blocks (HBM bound),
//   K3  per-sphere self operator Y = E X on FP64 tensor cores (mma.sync f64, DMMA),
//       whose epilogue also adds the K1 and K2 results.
// Operator definition O6 of DESIGN.md (paper: P:130-136, P:423-426 treat it as a
// black box).  Kernels written for sm_100a; no tcgen05 kind supports f64, so K3
// uses the DMMA path (measured 37.2 TFLOP/s on B200, same as DFMA).
#include <algorithm>

#include "bpqn_internal.h"

namespace bpqn {

static const double PI_D = 3.14159265358979323846;

// ------------------------------------------------------------------ K1
// Work item = (source chunk, target block).  A CTA of K1T threads owns K1R targets
// per thread; sources are staged in shared memory TS at a time, pre-folded with
// their weight and kernel constant.  Results are added with fp64 atomics (a
// handful of chunks per target).
constexpr int K1T = 128;
constexpr int K1R = 2;
constexpr int K1TS = 128;

__device__ __forceinline__ double rsqrt_f64(double x) {
  double y;
  asm("rsqrt.approx.f64 %0, %1;" : "=d"(y) : "d"(x));  // MUFU.RSQ64H + cubic refinement (ptxas)
  return y;
}

struct K1Args {
  const double* X;      // [N][3] targets
  const double* src;    // [N][8] {y, w, n, 0}
  const double* sigS;   // [N][3] single-layer density (S / SD modes)
  const double* sigD;   // [N][3] double-layer density (D / SD modes)
  double* out;          // [N][3] (atomic accumulate)
  int N;
  int n_tblocks, n_chunks, chunk;
  double cS, cD;
};

template <int MODE>
__global__ void __launch_bounds__(K1T, 4) k1_allpairs(K1Args A) {
  // per-source smem record: D: y(3) n(3) q~(3) ; S: y(3) f~(3) ; SD: y n f~ q~
  constexpr int REC = (MODE == MODE_D) ? 9 : (MODE == MODE_S ? 6 : 12);
  __shared__ double sh[K1TS * REC];
  const int n_items = A.n_tblocks * A.n_chunks;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int ch = item / A.n_tblocks;
    const int tb = item - ch * A.n_tblocks;
    double x[K1R][3], u[K1R][3];
#pragma unroll
    for (int r = 0; r < K1R; ++r) {
      int t = tb * (K1T * K1R) + r * K1T + threadIdx.x;
      int tc = t < A.N ? t : A.N - 1;
      x[r][0] = A.X[3 * tc];
      x[r][1] = A.X[3 * tc + 1];
      x[r][2] = A.X[3 * tc + 2];
      u[r][0] = u[r][1] = u[r][2] = 0.0;
    }
    const int s_begin = ch * A.chunk;
    const int s_end = min(A.N, s_begin + A.chunk);
    for (int s0 = s_begin; s0 < s_end; s0 += K1TS) {
      __syncthreads();
      for (int k = threadIdx.x; k < K1TS; k += K1T) {
        int j = s0 + k;
        double* rec = sh + k * REC;
        if (j < s_end) {
          const double* g = A.src + 8 * (size_t)j;
          double y0 = g[0], y1 = g[1], y2 = g[2], w = g[3];
          rec[0] = y0; rec[1] = y1; rec[2] = y2;
          if (MODE == MODE_D) {
            double c = A.cD * w;
            rec[3] = g[4]; rec[4] = g[5]; rec[5] = g[6];
            rec[6] = c * A.sigD[3 * j]; rec[7] = c * A.sigD[3 * j + 1]; rec[8] = c * A.sigD[3 * j + 2];
          } else if (MODE == MODE_S) {
            double c = A.cS * w;
            rec[3] = c * A.sigS[3 * j]; rec[4] = c * A.sigS[3 * j + 1]; rec[5] = c * A.sigS[3 * j + 2];
          } else {
            double c = A.cS * w, d = A.cD * w;
            rec[3] = g[4]; rec[4] = g[5]; rec[5] = g[6];
            rec[6] = c * A.sigS[3 * j]; rec[7] = c * A.sigS[3 * j + 1]; rec[8] = c * A.sigS[3 * j + 2];
            rec[9] = d * A.sigD[3 * j]; rec[10] = d * A.sigD[3 * j + 1]; rec[11] = d * A.sigD[3 * j + 2];
          }
        } else {
          rec[0] = rec[1] = rec[2] = 1e30;  // far away, zero strength
          for (int q = 3; q < REC; ++q) rec[q] = 0.0;
        }
      }
      __syncthreads();
      const int ns = K1TS;
#pragma unroll 2
      for (int k = 0; k < ns; ++k) {
        const double* rec = sh + k * REC;
        const double y0 = rec[0], y1 = rec[1], y2 = rec[2];
#pragma unroll
        for (int r = 0; r < K1R; ++r) {
          const double r0 = x[r][0] - y0, r1 = x[r][1] - y1, r2 = x[r][2] - y2;
          const double rr = fma(r2, r2, fma(r1, r1, r0 * r0));
          double s = rsqrt_f64(rr);
          s = (__double2hiint(rr) != 0) ? s : 0.0;  // the target's own node: rho = 0
          if (MODE == MODE_D) {
            const double rn = fma(r2, rec[5], fma(r1, rec[4], r0 * rec[3]));
            const double rq = fma(r2, rec[8], fma(r1, rec[7], r0 * rec[6]));
            const double s2 = s * s;
            double t = rn * rq;
            t = t * s2;
            t = t * s2;
            t = t * s;
            u[r][0] = fma(r0, t, u[r][0]);
            u[r][1] = fma(r1, t, u[r][1]);
            u[r][2] = fma(r2, t, u[r][2]);
          } else if (MODE == MODE_S) {
            const double f0 = rec[3], f1 = rec[4], f2 = rec[5];
            const double rf = fma(r2, f2, fma(r1, f1, r0 * f0));
            const double s3 = s * s * s;
            const double t = rf * s3;
            u[r][0] = fma(f0, s, fma(r0, t, u[r][0]));
            u[r][1] = fma(f1, s, fma(r1, t, u[r][1]));
            u[r][2] = fma(f2, s, fma(r2, t, u[r][2]));
          } else {
            const double rn = fma(r2, rec[5], fma(r1, rec[4], r0 * rec[3]));
            const double f0 = rec[6], f1 = rec[7], f2 = rec[8];
            const double rf = fma(r2, f2, fma(r1, f1, r0 * f0));
            const double rq = fma(r2, rec[11], fma(r1, rec[10], r0 * rec[9]));
            const double s2 = s * s;
            const double s3 = s2 * s;
            const double s5 = s3 * s2;
            const double t = fma(rf, s3, (rn * rq) * s5);
            u[r][0] = fma(f0, s, fma(r0, t, u[r][0]));
            u[r][1] = fma(f1, s, fma(r1, t, u[r][1]));
            u[r][2] = fma(f2, s, fma(r2, t, u[r][2]));
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < K1R; ++r) {
      int t = tb * (K1T * K1R) + r * K1T + threadIdx.x;
      if (t < A.N) {
        atomicAdd(A.out + 3 * t, u[r][0]);
        atomicAdd(A.out + 3 * t + 1, u[r][1]);
        atomicAdd(A.out + 3 * t + 2, u[r][2]);
      }
    }
  }
}

// Algorithmic flops per target-source pair of the fused formulation (DESIGN.md
// "Roofline"): S 28, D 29, S+D 42 (the rsqrt counted as one operation).
double allpairs_flops_per_pair(int mode) { return mode == MODE_S ? 28.0 : (mode == MODE_D ? 29.0 : 42.0); }

void launch_allpairs(Geom& g, int mode, const double* sigS, const double* sigD, double* out, cudaStream_t st) {
  K1Args A;
  A.X = g.X.p;
  A.src = g.src.p;
  A.sigS = sigS;
  A.sigD = sigD;
  A.out = out;
  A.N = g.n;
  A.n_tblocks = (g.n + K1T * K1R - 1) / (K1T * K1R);
  // chunking: enough items to fill the GPU several times over, chunk a multiple of K1TS
  const int resident = g.sms * 4;
  int want_chunks = std::max(1, (8 * resident + A.n_tblocks - 1) / A.n_tblocks);
  int chunk = (g.n + want_chunks - 1) / want_chunks;
  chunk = std::max(K1TS, ((chunk + K1TS - 1) / K1TS) * K1TS);
  A.chunk = chunk;
  A.n_chunks = (g.n + chunk - 1) / chunk;
  A.cS = 1.0 / (8.0 * PI_D * g.mu);
  A.cD = -3.0 / (4.0 * PI_D);
  int items = A.n_tblocks * A.n_chunks;
  int grid = std::min(items, resident);
  BPQN_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * 3 * (size_t)g.n, st));
  if (mode == MODE_D) k1_allpairs<MODE_D><<<grid, K1T, 0, st>>>(A);
  else if (mode == MODE_S) k1_allpairs<MODE_S><<<grid, K1T, 0, st>>>(A);
  else k1_allpairs<MODE_SD><<<grid, K1T, 0, st>>>(A);
  BPQN_CHECK_LAUNCH();
  g.prof.allpairs_launches++;
  g.prof.launches++;
}

// ------------------------------------------------------------------ K2
// One warp per (near target, component a): sum over the target's incidences of
// dot(M[inc][a][:], sigma_m[:]) (length 3nq).  Deterministic, no atomics.
__global__ void k2_near(int n_targets, const int* nt_list, const int* nt_ptr, const int* inc_m, int nq,
                        const double* MS, const double* sigS, const double* MD, const double* sigD, double* out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= 3 * n_targets) return;
  const int tix = warp / 3, a = warp - 3 * tix;
  const int i = nt_list[tix];
  const size_t len = 3 * (size_t)nq;
  double acc = 0.0;
  for (int k = nt_ptr[tix]; k < nt_ptr[tix + 1]; ++k) {
    const int m = inc_m[k];
    const size_t base = ((size_t)k * 3 + a) * len;
    if (MD) {
      const double* row = MD + base;
      const double* sg = sigD + (size_t)m * len;
      for (size_t c = lane; c < len; c += 32) acc = fma(__ldg(row + c), sg[c], acc);
    }
    if (MS) {
      const double* row = MS + base;
      const double* sg = sigS + (size_t)m * len;
      for (size_t c = lane; c < len; c += 32) acc = fma(__ldg(row + c), sg[c], acc);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) out[3 * (size_t)i + a] = acc;
}

void launch_near(Geom& g, const double* sigS, const double* sigD, double* out, cudaStream_t st) {
  BPQN_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * 3 * (size_t)g.n, st));
  g.prof.launches++;
  if (g.n_near_targets == 0) return;
  const double* MS = (sigS && g.M_S.p) ? g.M_S.p : nullptr;
  const double* MD = sigD ? g.M_D.p : nullptr;
  int warps = 3 * g.n_near_targets;
  int threads = 256;
  int blocks = (warps * 32 + threads - 1) / threads;
  k2_near<<<blocks, threads, 0, st>>>(g.n_near_targets, g.nt_list.p, g.nt_ptr.p, g.inc_m.p, g.nq, MS, sigS, MD,
                                      sigD, out);
  BPQN_CHECK_LAUNCH();
  g.prof.launches++;
}

// ------------------------------------------------------------------ K3
// C[M x Np] (column n = sphere n, contiguous M = 3nq) = E[M x M] * X[M x Np] (+ adds).
// CTA tile 64 x 32, K step 16, 4 warps of 32 x 16 each, mma.sync m8n8k4 f64 (DMMA).
constexpr int GBM = 64, GBN = 32, GBK = 16;

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(128) k3_self_gemm(int M, int Nn, const double* __restrict__ E,
                                                    const double* __restrict__ X, const double* add1,
                                                    const double* add2, double* out, int accumulate) {
  __shared__ double As[GBM][GBK + 1];
  __shared__ double Bs[GBN][GBK + 1];
  const int m0 = blockIdx.x * GBM, n0 = blockIdx.y * GBN;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 16;
  const int g = lane >> 2, t4 = lane & 3;
  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int k0 = 0; k0 < M; k0 += GBK) {
    __syncthreads();
    for (int e = threadIdx.x; e < GBM * GBK; e += 128) {
      int r = e / GBK, c = e - r * GBK;
      int gr = m0 + r, gc = k0 + c;
      As[r][c] = (gr < M && gc < M) ? E[(size_t)gr * M + gc] : 0.0;
    }
    for (int e = threadIdx.x; e < GBN * GBK; e += 128) {
      int nn = e / GBK, c = e - nn * GBK;
      int gn = n0 + nn, gc = k0 + c;
      Bs[nn][c] = (gn < Nn && gc < M) ? X[(size_t)gn * M + gc] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < GBK; kk += 4) {
      double af[4], bf[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = As[wm + 8 * i + g][kk + t4];
#pragma unroll
      for (int j = 0; j < 2; ++j) bf[j] = Bs[wn + 8 * j + g][kk + t4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  // epilogue: C fragment row = g, cols = 2*t4 + {0,1}
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        int row = m0 + wm + 8 * i + g;
        int col = n0 + wn + 8 * j + 2 * t4 + h;
        if (row < M && col < Nn) {
          size_t o = (size_t)col * M + row;
          double v = acc[i][j][h];
          if (add1) v += add1[o];
          if (add2) v += add2[o];
          if (accumulate) v += out[o];
          out[o] = v;
        }
      }
}

void launch_self_gemm(Geom& g, const double* E, const double* X, const double* add1, const double* add2,
                      double* out, int accumulate, cudaStream_t st) {
  int M = 3 * g.nq;
  dim3 grid((M + GBM - 1) / GBM, (g.np + GBN - 1) / GBN);
  k3_self_gemm<<<grid, 128, 0, st>>>(M, g.np, E, X, add1, add2, out, accumulate);
  BPQN_CHECK_LAUNCH();
  g.prof.launches++;
}

// ------------------------------------------------------------------ operator
// out = coarse all-pairs + near corrections + self blocks, for densities sigS
// (single layer, self matrix Es) and sigD (double layer, self matrix Ed).
void apply_operator(Geom& g, const double* sigS, const double* sigD, const double* Es, const double* Ed,
                    double* out, cudaStream_t st) {
  int mode = (sigS && sigD) ? MODE_SD : (sigS ? MODE_S : MODE_D);
  Profile& P = g.prof;
  cudaEvent_t* ev = nullptr;
  if (P.events) {
    while (P.pool.size() < P.used + 4) {
      cudaEvent_t e;
      BPQN_CUDA(cudaEventCreate(&e));
      P.pool.push_back(e);
    }
    ev = P.pool.data() + P.used;
    P.used += 4;
    BPQN_CUDA(cudaEventRecord(ev[0], st));
  }
  launch_allpairs(g, mode, sigS, sigD, g.far.p, st);
  if (ev) {
    BPQN_CUDA(cudaEventRecord(ev[1], st));
    P.allpairs_flop += (double)g.n * (double)g.n * allpairs_flops_per_pair(mode);
  }
  launch_near(g, sigS, sigD, g.nearout.p, st);
  if (ev) BPQN_CUDA(cudaEventRecord(ev[2], st));
  if (sigS && sigD) {
    launch_self_gemm(g, Es, sigS, g.far.p, g.nearout.p, out, 0, st);
    launch_self_gemm(g, Ed, sigD, nullptr, nullptr, out, 1, st);
  } else if (sigS) {
    launch_self_gemm(g, Es, sigS, g.far.p, g.nearout.p, out, 0, st);
  } else {
    launch_self_gemm(g, Ed, sigD, g.far.p, g.nearout.p, out, 0, st);
  }
  if (ev) BPQN_CUDA(cudaEventRecord(ev[3], st));
}

// Sum the recorded operator timings (one host sync) and recycle the events.
void profile_collect(Geom& g) {
  Profile& P = g.prof;
  if (P.used == 0) return;
  BPQN_CUDA(cudaEventSynchronize(P.pool[P.used - 1]));
  for (size_t k = 0; k < P.used; k += 4) {
    float a = 0, b = 0, c = 0;
    BPQN_CUDA(cudaEventElapsedTime(&a, P.pool[k], P.pool[k + 1]));
    BPQN_CUDA(cudaEventElapsedTime(&b, P.pool[k + 1], P.pool[k + 2]));
    BPQN_CUDA(cudaEventElapsedTime(&c, P.pool[k + 2], P.pool[k + 3]));
    P.ms_allpairs += a;
    P.ms_near += b;
    P.ms_self += c;
  }
  P.used = 0;
}

}  // namespace bpqn
