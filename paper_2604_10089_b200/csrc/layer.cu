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
// dot(M[inc][a][:], sigma_m[:]) (length 3nq, even).  The correction rows stream from
// HBM exactly once per apply (16-byte streaming loads, 4 in flight per lane); the
// densities are L2-resident.  Deterministic, no atomics.
__device__ __forceinline__ double dot_row(const double* __restrict__ row, const double* __restrict__ sg, int len2,
                                          int lane, double acc) {
  const double2* r2 = reinterpret_cast<const double2*>(row);
  const double2* s2 = reinterpret_cast<const double2*>(sg);
  int c = lane;
  for (; c + 96 < len2; c += 128) {
    const double2 a0 = __ldcs(r2 + c), a1 = __ldcs(r2 + c + 32), a2 = __ldcs(r2 + c + 64), a3 = __ldcs(r2 + c + 96);
    const double2 b0 = __ldg(s2 + c), b1 = __ldg(s2 + c + 32), b2 = __ldg(s2 + c + 64), b3 = __ldg(s2 + c + 96);
    acc = fma(a0.x, b0.x, acc);
    acc = fma(a0.y, b0.y, acc);
    acc = fma(a1.x, b1.x, acc);
    acc = fma(a1.y, b1.y, acc);
    acc = fma(a2.x, b2.x, acc);
    acc = fma(a2.y, b2.y, acc);
    acc = fma(a3.x, b3.x, acc);
    acc = fma(a3.y, b3.y, acc);
  }
  for (; c < len2; c += 32) {
    const double2 a0 = __ldcs(r2 + c), b0 = __ldg(s2 + c);
    acc = fma(a0.x, b0.x, acc);
    acc = fma(a0.y, b0.y, acc);
  }
  return acc;
}

__global__ void k2_near(int n_targets, const int* nt_list, const int* nt_ptr, const int* inc_m, int nq,
                        const double* MS, const double* sigS, const double* MD, const double* sigD, double* out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= 3 * n_targets) return;
  const int tix = warp / 3, a = warp - 3 * tix;
  const int i = nt_list[tix];
  const size_t len = 3 * (size_t)nq;
  const int len2 = (int)(len / 2);
  double acc = 0.0;
  for (int k = nt_ptr[tix]; k < nt_ptr[tix + 1]; ++k) {
    const int m = inc_m[k];
    const size_t base = ((size_t)k * 3 + a) * len;
    if (MD) acc = dot_row(MD + base, sigD + (size_t)m * len, len2, lane, acc);
    if (MS) acc = dot_row(MS + base, sigS + (size_t)m * len, len2, lane, acc);
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
  // sharded: only this rank's near targets (the list is sorted by target node)
  const int k0 = g.shard_world > 1 ? g.sh_k0 : 0, k1 = g.shard_world > 1 ? g.sh_k1 : g.n_near_targets;
  if (k1 <= k0) return;
  int warps = 3 * (k1 - k0);
  int threads = 256;
  int blocks = (warps * 32 + threads - 1) / threads;
  k2_near<<<blocks, threads, 0, st>>>(k1 - k0, g.nt_list.p + k0, g.nt_ptr.p + k0, g.inc_m.p, g.nq, MS, sigS, MD,
                                      sigD, out);
  BPQN_CHECK_LAUNCH();
  g.prof.launches++;
}

// ------------------------------------------------------------------ K3
// C[M x Np] (column n = sphere n, contiguous M = 3nq) = E[M x M] X[M x Np], E row-major,
// the same for every sphere (translation invariance of the self rule).  FP64 tensor
// cores via mma.sync m8n8k4 (DMMA; tcgen05 has no f64 kind).  CTA tile 64 x 72
// (8 warps, each one 8-row strip x 9 n8 tiles), K in stages of 16 through a 3-deep
// cp.async ring (zero-filled tails), split-K over gridDim.z with fp64 atomics into an
// output that k3_prologue initialised with the fused additions (K1 + K2 results).
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

__global__ void k3_prologue(size_t n, const double* add1, const double* add2, double* out, int accumulate) {
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
    double v = accumulate ? out[e] : 0.0;
    if (add1) v += add1[e];
    if (add2) v += add2[e];
    out[e] = v;
  }
}

__global__ void __launch_bounds__(256) k3_self_gemm(int M, int Nn, int kchunk, const double* __restrict__ E,
                                                    const double* __restrict__ X, double* out) {
  extern __shared__ __align__(16) double k3_dyn[];
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
  if (row < M) {
#pragma unroll
    for (int j = 0; j < 9; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = n0 + j * 8 + 2 * t4 + h;
        if (col < Nn) atomicAdd(out + (size_t)col * M + row, acc[j][h]);
      }
  }
}

void launch_self_gemm(Geom& g, const double* E, const double* X, const double* add1, const double* add2,
                      double* out, int accumulate, cudaStream_t st, int s0, int s1) {
  // spheres [s0, s1) only (sharded operator); columns are contiguous per sphere
  if (s1 < 0) s1 = g.np;
  const int M = 3 * g.nq, ncol = s1 - s0;
  if (ncol <= 0) return;
  const size_t off = (size_t)M * s0;
  X += off;
  out += off;
  if (add1) add1 += off;
  if (add2) add2 += off;
  const size_t n = (size_t)M * ncol;
  k3_prologue<<<(unsigned)std::min<size_t>((n + 255) / 256, 4 * (size_t)g.sms), 256, 0, st>>>(n, add1, add2, out,
                                                                                            accumulate);
  const int mt = (M + K3_BM - 1) / K3_BM, nt = (ncol + K3_BN - 1) / K3_BN;
  // split K so that the grid covers the GPU about twice; no split (a single writer per
  // output, bit-reproducible) when sharded, so that every rank's replicated GMRES agrees
  int ks = std::max(1, std::min((2 * g.sms + mt * nt - 1) / (mt * nt), (M + 8 * K3_BK - 1) / (8 * K3_BK)));
  if (g.shard_world > 1) ks = 1;
  int kchunk = (M + ks - 1) / ks;
  kchunk = ((kchunk + K3_BK - 1) / K3_BK) * K3_BK;
  ks = (M + kchunk - 1) / kchunk;
  dim3 grid(mt, nt, ks);
  static bool attr = false;
  if (!attr) {
    BPQN_CUDA(cudaFuncSetAttribute(k3_self_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, K3_SMEM));
    attr = true;
  }
  k3_self_gemm<<<grid, 256, K3_SMEM, st>>>(M, ncol, kchunk, E, X, out);
  BPQN_CHECK_LAUNCH();
  g.prof.launches += 2;
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

static void shard_exchange(Geom& g, double* out, cudaStream_t st) {
  const int nrow = g.sh_t1 - g.sh_t0;
  k_shard_pack<<<(3 * g.sh_rows + 255) / 256, 256, 0, st>>>(out, g.sh_t0, nrow, g.sh_send, g.sh_rows);
  BPQN_CHECK_LAUNCH();
  BPQN_CUDA(cudaStreamSynchronize(st));
  if (g.sh_fn(g.sh_user) != 0) throw Error{BPQN_ERR_CUDA, "shard all-gather callback failed"};
  const long long tot = 3LL * g.sh_rows * g.shard_world;
  k_shard_unpack<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(g.sh_recv, g.shard_world, g.sh_rows, g.np, g.nq, out);
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
  const bool overlap = g.overlap_k2;
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
  if (overlap) {
    BPQN_CUDA(cudaEventRecord(g.ev_fork, st));
    BPQN_CUDA(cudaStreamWaitEvent(g.side, g.ev_fork, 0));
  }
  if (ev) BPQN_CUDA(cudaEventRecord(ev[2], sk2));
  launch_near(g, sigS, sigD, g.nearout.p, sk2);
  if (ev) BPQN_CUDA(cudaEventRecord(ev[3], sk2));
  if (ev) BPQN_CUDA(cudaEventRecord(ev[0], st));
  launch_allpairs(g, mode, sigS, sigD, g.far.p, st);
  if (ev) {
    BPQN_CUDA(cudaEventRecord(ev[1], st));
    const double ntg = g.shard_world > 1 ? (double)(g.sh_t1 - g.sh_t0) : (double)g.n;  // this rank's targets
    P.allpairs_flop += (double)g.n * ntg * allpairs_flops_per_pair(mode);
  }
  if (overlap) {
    BPQN_CUDA(cudaEventRecord(g.ev_join, g.side));
    BPQN_CUDA(cudaStreamWaitEvent(st, g.ev_join, 0));
  }
  const bool sharded = g.shard_world > 1;
  const int s0 = sharded ? g.sh_s0 : 0, s1 = sharded ? g.sh_s1 : g.np;
  if (sigS && sigD) {
    launch_self_gemm(g, Es, sigS, g.far.p, g.nearout.p, out, 0, st, s0, s1);
    launch_self_gemm(g, Ed, sigD, nullptr, nullptr, out, 1, st, s0, s1);
  } else if (sigS) {
    launch_self_gemm(g, Es, sigS, g.far.p, g.nearout.p, out, 0, st, s0, s1);
  } else {
    launch_self_gemm(g, Ed, sigD, g.far.p, g.nearout.p, out, 0, st, s0, s1);
  }
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
