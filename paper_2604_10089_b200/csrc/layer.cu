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
