// K1: all-pairs coarse-rule Stokeslet / stresslet summation on B200 (sm_100a).
//
//   u(x_i) = sum_{j != i} w_j [ G(x_i - y_j) f_j + K_D(x_i, y_j) q_j ]      (O6, coarse part)
//   G(r)   = (I/rho + r r^T/rho^3) / (8 pi mu),   K_D = -3/(4 pi) (r.n_y) r r^T / rho^5,  r = x - y
//
// over ALL node pairs with rho > 0 (the same-sphere and near-pair coarse terms are
// removed again by K3's E matrices and K2's correction blocks).  The paper treats
// this operator as a black box (STKFMM far field
// P:528); the B200 design is DESIGN.md "K1":
//
//  * k1_pack writes the sources once per call as 16-byte-aligned records with the
//    weight and kernel constant folded into the density (S: y, f~; D: y, n, q~;
//    S+D: y, n, f~, q~), padded to a whole number of source tiles with far-away
//    zero-strength records -- the main loop has no bounds checks.
//  * k1_allpairs is persistent: the (target block, source tile) work space is cut
//    into equal contiguous ranges, one per resident CTA (perfect balance to one
//    tile, any N).  Source tiles stream through a K1_STAGES-deep shared-memory ring
//    filled by one thread with TMA bulk copies (cp.async.bulk + mbarrier
//    complete_tx); all threads read them back as broadcast 16-byte loads.
//  * each thread owns K1_R targets in registers; a target block's partial sums are
//    stored as partial sums when the CTA's range leaves the block (one segment per (CTA, block)),
//    added in a fixed order by k_row_reduce (no floating-point atomics: bit-reproducible).
//  * rho^-k from one MUFU.RSQ64H seed y (rsqrt.approx.ftz.f64) and the series
//    (1-e)^(-k/2) = 1 + (k/2) e + (k/2)(k/2+1)/2 e^2, e = 1 - rho^2 y^2 (|e| <= 1.85e-6
//    = 2^-19 measured, tools/rsq_micro.cu; truncation error < 7|e|^3 ~ 4e-17): rho^-5 costs
//    6 FP64 instructions instead of the 9 of rsqrt() + powers.  rho = 0 (the target's
//    own node) zeroes the seed with an integer select, so that pair contributes 0.
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "bpqn_internal.h"

namespace bpqn {

static const double PI_A = 3.14159265358979323846;

constexpr int K1_THREADS = 256;
constexpr int K1_R = 4;                          // targets per thread
constexpr int K1_TB = K1_THREADS * K1_R;         // targets per block
constexpr int K1_TS = 64;                        // sources per tile
constexpr int K1_STAGES = 4;                     // smem ring depth

template <int MODE>
struct Rec;
template <>
struct Rec<MODE_S> { static constexpr int n = 6; };    // y0 y1 y2 f0 f1 f2
template <>
struct Rec<MODE_D> { static constexpr int n = 10; };   // y0 y1 y2 n0 n1 n2 q0 q1 q2 pad
template <>
struct Rec<MODE_SD> { static constexpr int n = 14; };  // y0 y1 y2 n0 n1 n2 f0 f1 f2 q0 q1 q2 pad pad

__global__ void k1_pack(int mode, int N, int npad, const double* __restrict__ src, const double* __restrict__ sigS,
                        const double* __restrict__ sigD, double cS, double cD, double* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= npad) return;
  const int rec = mode == MODE_S ? 6 : (mode == MODE_D ? 10 : 14);
  double* o = out + (size_t)rec * j;
  if (j >= N) {  // far away, zero strength
    o[0] = o[1] = o[2] = 1e30;
    for (int k = 3; k < rec; ++k) o[k] = 0.0;
    return;
  }
  const double* g = src + 8 * (size_t)j;  // {y, w, n, 0}
  const double w = g[3];
  o[0] = g[0];
  o[1] = g[1];
  o[2] = g[2];
  if (mode == MODE_S) {
    const double c = cS * w;
    o[3] = c * sigS[3 * (size_t)j];
    o[4] = c * sigS[3 * (size_t)j + 1];
    o[5] = c * sigS[3 * (size_t)j + 2];
  } else {
    o[3] = g[4];
    o[4] = g[5];
    o[5] = g[6];
    if (mode == MODE_D) {
      const double c = cD * w;
      o[6] = c * sigD[3 * (size_t)j];
      o[7] = c * sigD[3 * (size_t)j + 1];
      o[8] = c * sigD[3 * (size_t)j + 2];
      o[9] = 0.0;
    } else {
      const double c = cS * w, d = cD * w;
      o[6] = c * sigS[3 * (size_t)j];
      o[7] = c * sigS[3 * (size_t)j + 1];
      o[8] = c * sigS[3 * (size_t)j + 2];
      o[9] = d * sigD[3 * (size_t)j];
      o[10] = d * sigD[3 * (size_t)j + 1];
      o[11] = d * sigD[3 * (size_t)j + 2];
      o[12] = o[13] = 0.0;
    }
  }
}

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "LAB_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra LAB_WAIT_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ double rsq_seed(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));  // one MUFU.RSQ64H
  return y;
}

__device__ __forceinline__ double lds_f64(unsigned addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}

// seed y ~ rr^-1/2 with rr == 0 -> y = 0 (integer select, no FP64 compare)
__device__ __forceinline__ double seed_or_zero(double rr) {
  const double y = rsq_seed(rr);
  const int hi = __double2hiint(rr) != 0 ? __double2hiint(y) : 0;
  return __hiloint2double(hi, __double2hiint(rr) != 0 ? __double2loint(y) : 0);
}

struct K1Params {
  const double* X;     // [N][3] node positions (targets t0 .. t0 + nt - 1)
  const double* pk;    // packed sources [npad][REC]
  double* pseg;        // [grid + n_tb][K1_TB][3]: CTA c's sums over target block tb at segment c + tb
  int t0, nt, n_tb, n_st;
  long long units;     // n_tb * n_st
};

template <int MODE>
__global__ void __launch_bounds__(K1_THREADS, 2) k1_allpairs(K1Params P) {
  constexpr int REC = Rec<MODE>::n;
  constexpr int TILE_DBL = K1_TS * REC;
  constexpr unsigned TILE_BYTES = TILE_DBL * 8;
  __shared__ __align__(128) double ring[K1_STAGES][TILE_DBL];
  __shared__ __align__(8) uint64_t full[K1_STAGES];

  const long long P_ = gridDim.x;
  const long long u0 = P.units * blockIdx.x / P_;
  const long long u1 = P.units * (blockIdx.x + 1) / P_;
  const int tid = threadIdx.x;
  if (u0 >= u1) return;

  if (tid == 0) {
    for (int s = 0; s < K1_STAGES; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < K1_STAGES && u0 + s < u1; ++s) {
      const long long u = u0 + s;
      const int st = (int)(u % P.n_st);
      mbar_expect_tx(&full[s], TILE_BYTES);
      bulk_g2s(ring[s], P.pk + (size_t)st * TILE_DBL, TILE_BYTES, &full[s]);
    }
  }

  double x[K1_R][3], acc[K1_R][3];
  int cur_tb = -1;
  for (long long u = u0; u < u1; ++u) {
    const int i = (int)(u - u0);
    const int buf = i % K1_STAGES;
    const unsigned parity = (unsigned)(i / K1_STAGES) & 1u;
    const int tb = (int)(u / P.n_st);
    if (tb != cur_tb) {
      if (cur_tb >= 0) {  // segment blockIdx.x + cur_tb (fixed-order sum in k_row_reduce)
        double* sg = P.pseg + (size_t)(blockIdx.x + cur_tb) * K1_TB * 3;
#pragma unroll
        for (int r = 0; r < K1_R; ++r) {
          const int lr = r * K1_THREADS + tid;
          sg[3 * lr] = acc[r][0];
          sg[3 * lr + 1] = acc[r][1];
          sg[3 * lr + 2] = acc[r][2];
        }
      }
      cur_tb = tb;
#pragma unroll
      for (int r = 0; r < K1_R; ++r) {
        int tl = tb * K1_TB + r * K1_THREADS + tid;
        const int t = P.t0 + (tl < P.nt ? tl : P.nt - 1);
        x[r][0] = P.X[3 * (size_t)t];
        x[r][1] = P.X[3 * (size_t)t + 1];
        x[r][2] = P.X[3 * (size_t)t + 2];
        acc[r][0] = acc[r][1] = acc[r][2] = 0.0;
      }
    }
    mbar_wait(&full[buf], parity);
    const double* tile = ring[buf];
#pragma unroll 2
    for (int k = 0; k < K1_TS; ++k) {
      const double2* rp = reinterpret_cast<const double2*>(tile + k * REC);
      double src[REC];
#pragma unroll
      for (int h = 0; h < REC / 2; ++h) {
        const double2 v = rp[h];
        src[2 * h] = v.x;
        src[2 * h + 1] = v.y;
      }
#pragma unroll
      for (int r = 0; r < K1_R; ++r) {
        const double r0 = x[r][0] - src[0], r1 = x[r][1] - src[1], r2 = x[r][2] - src[2];
        const double rr = fma(r2, r2, fma(r1, r1, r0 * r0));
        const double y = seed_or_zero(rr);
        const double y2 = y * y;
        const double e = fma(-rr, y2, 1.0);
        if (MODE == MODE_D) {
          // rho^-5 = y^5 (1 + 5/2 e + 35/8 e^2)
          const double rn = fma(r2, src[5], fma(r1, src[4], r0 * src[3]));
          const double rq = fma(r2, src[8], fma(r1, src[7], r0 * src[6]));
          const double c5 = fma(e, fma(e, 4.375, 2.5), 1.0);
          const double y4 = y2 * y2;
          double t = rn * rq;
          t = t * y;
          t = t * y4;
          t = t * c5;
          acc[r][0] = fma(r0, t, acc[r][0]);
          acc[r][1] = fma(r1, t, acc[r][1]);
          acc[r][2] = fma(r2, t, acc[r][2]);
        } else {
          // rho^-1 = y (1 + e/2 + 3/8 e^2)
          const double s = fma(y * e, fma(e, 0.375, 0.5), y);
          const double s2 = s * s;
          const double s3 = s2 * s;
          if (MODE == MODE_S) {
            const double rf = fma(r2, src[5], fma(r1, src[4], r0 * src[3]));
            const double t = rf * s3;
            acc[r][0] = fma(src[3], s, fma(r0, t, acc[r][0]));
            acc[r][1] = fma(src[4], s, fma(r1, t, acc[r][1]));
            acc[r][2] = fma(src[5], s, fma(r2, t, acc[r][2]));
          } else {
            const double rn = fma(r2, src[5], fma(r1, src[4], r0 * src[3]));
            const double rf = fma(r2, src[8], fma(r1, src[7], r0 * src[6]));
            const double rq = fma(r2, src[11], fma(r1, src[10], r0 * src[9]));
            const double s5 = s3 * s2;
            const double t = fma(rf, s3, (rn * rq) * s5);
            acc[r][0] = fma(src[6], s, fma(r0, t, acc[r][0]));
            acc[r][1] = fma(src[7], s, fma(r1, t, acc[r][1]));
            acc[r][2] = fma(src[8], s, fma(r2, t, acc[r][2]));
          }
        }
      }
    }
    __syncthreads();  // every thread is done with ring[buf]
    if (tid == 0 && u + K1_STAGES < u1) {
      const int st = (int)((u + K1_STAGES) % P.n_st);
      mbar_expect_tx(&full[buf], TILE_BYTES);
      bulk_g2s(ring[buf], P.pk + (size_t)st * TILE_DBL, TILE_BYTES, &full[buf]);
    }
  }
  {
    double* sg = P.pseg + (size_t)(blockIdx.x + cur_tb) * K1_TB * 3;
#pragma unroll
    for (int r = 0; r < K1_R; ++r) {
      const int lr = r * K1_THREADS + tid;
      sg[3 * lr] = acc[r][0];
      sg[3 * lr + 1] = acc[r][1];
      sg[3 * lr + 2] = acc[r][2];
    }
  }
}

// ---------------------------------------------------------------- symmetric K1
// Newton's third law: every unordered pair {i, j} of distinct blocks is evaluated
// once and contributes to both u_i and u_j, sharing r, rho^2 and the rho^-k powers
// (D mode: 35 FP64 instructions per pair = 17.5 per interaction, vs 24 above).
//  * points are cut into blocks of KS_B = 32 R KS_W; a CTA holds one block as
//    targets (R per lane, with their own n / f~ / q~ for the reverse direction);
//  * work units (block b, 64-point source tile t) with t >= the block's first tile;
//    tiles inside the block ("diagonal") run the one-directional loop, later tiles
//    the symmetric one -- each unordered pair is covered exactly once;
//  * symmetric loop per 32-point group: at step k lane l evaluates source
//    (l + k) mod 32 (lane-distinct, conflict-free LDS.128 from the TMA ring) and
//    carries that source's accumulator, which rotates one lane per step by
//    __shfl_sync; after 32 steps lane l holds source l's sum.  The 8 warps' sums
//    are reduced through shared memory and stored as the unit's source-side partial sums.
//  * sources are points of spheres of radius a, so r.n_y = (h_m(x) - rho^2) / (2a) with
//    h_m(x) = |x - c_m|^2 - a^2 per (target, source sphere): the forward r.n costs one FMA
//    and the records carry no normals.  A 32-point source group spans at most two spheres
//    (Nq >= 32 is checked), so each target keeps h for both (recomputed when the group's first
//    sphere changes).
struct K1SymParams {
  const double* pk;       // packed records [npad][RecS] (targets and sources)
  const double* centers;  // [Np][3]
  // deterministic partial sums (no atomics; k_row_reduce adds them in a fixed order):
  double* pseg;           // [grid + nb][KS_B][3]: target-side sums of CTA c over block b at segment c + b
  double* psrc;           // [nb][psrc_ld]: source-side sums of unit (b, t) at psrc[b][3 (64 t + j) + comp]
  size_t psrc_ld;
  int N, nb, nt, nq, np;  // blocks of KS_B points, tiles of K1_TS points, nodes per sphere, spheres
  double a;
  long long units;        // units this launch processes: [ubeg, ubeg + units) of the block-major list
  long long ubeg;         // (ubeg > 0 only when sharded over ranks, bpqn_geometry_shard_symmetric)
};

// compact records of the symmetric kernel: S {y, f~}, D {y, q~}, S+D {y, f~, q~, pad}
template <int MODE>
struct RecS { static constexpr int n = MODE == MODE_S ? 6 : (MODE == MODE_D ? 6 : 10); };
// per-target registers: x and its own density (the record without padding); the reverse
// stresslet's r.n_t comes from the sphere identity via H (see k1_sym)
template <int MODE>
struct TgtN { static constexpr int n = MODE == MODE_SD ? 9 : 6; };

__global__ void k1_pack_sym(int mode, int N, int npad, const double* __restrict__ src,
                            const double* __restrict__ sigS, const double* __restrict__ sigD, double cS, double cD,
                            double* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= npad) return;
  const int rec = mode == MODE_SD ? 10 : 6;
  double* o = out + (size_t)rec * j;
  if (j >= N) {  // far away, zero strength
    o[0] = o[1] = o[2] = 1e30;
    for (int k = 3; k < rec; ++k) o[k] = 0.0;
    return;
  }
  const double* g = src + 8 * (size_t)j;  // {y, w, n, 0}
  const double w = g[3];
  o[0] = g[0];
  o[1] = g[1];
  o[2] = g[2];
  if (mode != MODE_D) {
    const double c = cS * w;
    o[3] = c * sigS[3 * (size_t)j];
    o[4] = c * sigS[3 * (size_t)j + 1];
    o[5] = c * sigS[3 * (size_t)j + 2];
  }
  if (mode != MODE_S) {
    const double d = cD * w;
    const int b = mode == MODE_D ? 3 : 6;
    o[b] = d * sigD[3 * (size_t)j];
    o[b + 1] = d * sigD[3 * (size_t)j + 1];
    o[b + 2] = d * sigD[3 * (size_t)j + 2];
  }
  if (mode == MODE_SD) o[9] = 0.0;
}

// One 32-source group.  tg[r] = {x(3), [f~(3)], [q~(3)]} (see TgtN / k1_sym);
// h[r][0|1] = (|x - c_m|^2 - a^2)/(2a) for the group's first / second source sphere,
// sources with in-tile index >= jb belong to the second; Hg[slot * 2 K1_TS + 64 g + u] (u < 64) =
// (|y_j - c_t|^2 - a^2)/(2a) for the block's target spheres (reverse r.n_t).
// SYM: off-diagonal tile, never a target's own node (rho > 0 for every pair, so the seed
// needs no zero mask: padded targets occur only in the last block, whose tiles are all
// diagonal).  MIXED: the group straddles the tile's sphere boundary (per-pair select of h);
// otherwise h is chosen once per group (always so at p = 16, where Nq = 17 x 32).
// TQ: the targets' own densities (record entries >= 3, used by the reverse direction only) live in
// shared memory (tq[c - 3][tq_stride], this lane's entry of target r at tq[(c - 3) tq_stride + 32 r])
// instead of registers -- fewer live registers per target, more room to interleave pair chains.
#define K1_TGV(r, c) (TQ ? tq[((c) - 3) * tq_stride + (r) * 32] : tg[r][c])
template <int MODE, int R, bool SYM, bool MIXED, int UNR, bool TQ>
__device__ __forceinline__ void k1_group(const double* __restrict__ gr, const double (&tg)[R][TgtN<MODE>::n],
                                         const double (&h)[R][2], int jl0, int jb, double inv2a,
                                         const double* __restrict__ Hg, const int (&slot)[R], double (&acc)[R][3],
                                         int lane, double& as0, double& as1, double& as2, const double* tq,
                                         int tq_stride) {
  constexpr int REC = RecS<MODE>::n;
  constexpr int QO = MODE == MODE_D ? 3 : 6;  // offset of q~ in a source record
  double hu[R];
  unsigned hb[R];  // shared address of this lane's window of the doubled H row: H(y_{(lane + k) & 31}) at hb + 8k
  const bool all_second = jl0 >= jb;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    hu[r] = all_second ? h[r][1] : h[r][0];
    hb[r] = smem_addr(Hg + slot[r] * (2 * K1_TS) + (jl0 >> 5) * 64 + lane);
  }
#pragma unroll UNR
  for (int k = 0; k < 32; ++k) {
    const int j = (lane + k) & 31;
    const double2* rp = reinterpret_cast<const double2*>(gr + j * REC);
    double sc[REC];
#pragma unroll
    for (int hh = 0; hh < REC / 2; ++hh) {
      const double2 v = rp[hh];
      sc[2 * hh] = v.x;
      sc[2 * hh + 1] = v.y;
    }
    const bool second = jl0 + j >= jb;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double r0 = tg[r][0] - sc[0], r1 = tg[r][1] - sc[1], r2 = tg[r][2] - sc[2];
      const double rr = fma(r2, r2, fma(r1, r1, r0 * r0));
      const double y = SYM ? rsq_seed(rr) : seed_or_zero(rr);
      const double y2 = y * y;
      const double e = fma(-rr, y2, 1.0);
      if (MODE == MODE_S) {
        const double s = fma(y * e, fma(e, 0.375, 0.5), y);
        const double s3 = (s * s) * s;
        const double rf = fma(r2, sc[5], fma(r1, sc[4], r0 * sc[3]));
        const double tf = rf * s3;
        acc[r][0] = fma(sc[3], s, fma(r0, tf, acc[r][0]));
        acc[r][1] = fma(sc[4], s, fma(r1, tf, acc[r][1]));
        acc[r][2] = fma(sc[5], s, fma(r2, tf, acc[r][2]));
        if (SYM) {  // G(-r) = G(r)
          const double rf2 = fma(r2, K1_TGV(r, 5), fma(r1, K1_TGV(r, 4), r0 * K1_TGV(r, 3)));
          const double tb = rf2 * s3;
          as0 = fma(K1_TGV(r, 3), s, fma(r0, tb, as0));
          as1 = fma(K1_TGV(r, 4), s, fma(r1, tb, as1));
          as2 = fma(K1_TGV(r, 5), s, fma(r2, tb, as2));
        }
      } else {
        const double hm = MIXED ? (second ? h[r][1] : h[r][0]) : hu[r];
        const double rq = fma(r2, sc[QO + 2], fma(r1, sc[QO + 1], r0 * sc[QO]));
        double s, s3, s5;
        if (MODE == MODE_D) {
          s5 = (y * (y2 * y2)) * fma(e, fma(e, 4.375, 2.5), 1.0);
          s = s3 = 0.0;
        } else {
          s = fma(y * e, fma(e, 0.375, 0.5), y);
          const double s2 = s * s;
          s3 = s2 * s;
          s5 = s3 * s2;
        }
        if (MODE == MODE_D) {
          // r.n kept scaled by 2a (h, H unscaled; the 1/(2a) is folded into q~ by
          // k1_pack_sym): 2a (r.n_y) rho^-5 = h s5 - rho^2 s5, one FMA per direction after the
          // shared c3 = rho^2 s5 (30 FP64 instructions per unordered pair instead of 31)
          const double c3 = rr * s5;
          const double tf = fma(hm, s5, -c3) * rq;
          acc[r][0] = fma(r0, tf, acc[r][0]);
          acc[r][1] = fma(r1, tf, acc[r][1]);
          acc[r][2] = fma(r2, tf, acc[r][2]);
          if (SYM) {  // K_D(x_j, y_i) q_i = -(r.n_i)(r.q_i) r / rho^5, 2a r.n_i = rho^2 - H
            const double rq2 = fma(r2, K1_TGV(r, 5), fma(r1, K1_TGV(r, 4), r0 * K1_TGV(r, 3)));
            const double tb = fma(-lds_f64(hb[r] + 8 * k), s5, c3) * rq2;
            as0 = fma(-r0, tb, as0);
            as1 = fma(-r1, tb, as1);
            as2 = fma(-r2, tb, as2);
          }
        } else {
          // as D mode: 2a r.n rho^-5 = h s5 - rho^2 s5 with rho^2 s5 = s3 (to rounding), q~ / (2a)
          const double rf = fma(r2, sc[5], fma(r1, sc[4], r0 * sc[3]));
          const double tf = fma(rf, s3, fma(hm, s5, -s3) * rq);
          acc[r][0] = fma(sc[3], s, fma(r0, tf, acc[r][0]));
          acc[r][1] = fma(sc[4], s, fma(r1, tf, acc[r][1]));
          acc[r][2] = fma(sc[5], s, fma(r2, tf, acc[r][2]));
          if (SYM) {
            const double rf2 = fma(r2, K1_TGV(r, 5), fma(r1, K1_TGV(r, 4), r0 * K1_TGV(r, 3)));
            const double rq2 = fma(r2, K1_TGV(r, 8), fma(r1, K1_TGV(r, 7), r0 * K1_TGV(r, 6)));
            const double tb = fma(rf2, s3, -(fma(-lds_f64(hb[r] + 8 * k), s5, s3) * rq2));
            as0 = fma(K1_TGV(r, 3), s, fma(r0, tb, as0));
            as1 = fma(K1_TGV(r, 4), s, fma(r1, tb, as1));
            as2 = fma(K1_TGV(r, 5), s, fma(r2, tb, as2));
          }
        }
      }
    }
    if (SYM) {  // the source accumulators travel with the sources: lane l takes lane l+1's
      const int from = (lane + 1) & 31;
      as0 = __shfl_sync(0xffffffffu, as0, from);
      as1 = __shfl_sync(0xffffffffu, as1, from);
      as2 = __shfl_sync(0xffffffffu, as2, from);
    }
  }
}

template <int MODE, int KS_W, int R, int MINB, int UNR, bool TQ = false>
__global__ void __launch_bounds__(32 * KS_W, MINB) k1_sym(K1SymParams P) {
  constexpr int REC = RecS<MODE>::n;
  constexpr int TN = TgtN<MODE>::n;
  constexpr int KS_B = 32 * R * KS_W;
  constexpr int TPB = KS_B / K1_TS;
  constexpr int TILE_DBL = K1_TS * REC;
  constexpr unsigned TILE_BYTES = TILE_DBL * 8;
  constexpr int NS = K1_STAGES;
  extern __shared__ __align__(128) double k1_dyn[];
  double (*ring)[TILE_DBL] = reinterpret_cast<double (*)[TILE_DBL]>(k1_dyn);            // [NS][TILE_DBL]
  double (*red)[KS_W][K1_TS * 3] =
      reinterpret_cast<double (*)[KS_W][K1_TS * 3]>(k1_dyn + NS * TILE_DBL);             // [2][W][192]
  double* tqs = k1_dyn + NS * TILE_DBL + 2 * KS_W * K1_TS * 3;                            // TQ: [TN-3][KS_B]
  double* cs = tqs + (TQ ? (TN - 3) * KS_B : 0);                                          // centres [Np][3]
  double* Hs = cs + (MODE == MODE_S ? 0 : 3 * P.np);                                      // [slots][2 K1_TS]
  __shared__ __align__(8) uint64_t full[NS];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long u0 = P.ubeg + P.units * blockIdx.x / gridDim.x;
  const long long u1 = P.ubeg + P.units * (blockIdx.x + 1) / gridDim.x;
  if (u0 >= u1) return;
  if (MODE != MODE_S)
    for (int e = tid; e < 3 * P.np; e += blockDim.x) cs[e] = P.centers[e];
  // unit u0 -> (block, tile); units run block-major, tiles from the block's first tile to the end
  int b_cur = 0;
  long long base = 0;
  while (base + (P.nt - b_cur * TPB) <= u0) {
    base += P.nt - b_cur * TPB;
    ++b_cur;
  }
  int t_cur = b_cur * TPB + (int)(u0 - base);
  int pb = b_cur, pt = t_cur;  // producer iterator (meaningful in thread 0 only)
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < NS && u0 + s < u1; ++s) {
      mbar_expect_tx(&full[s], TILE_BYTES);
      bulk_g2s(ring[s], P.pk + (size_t)pt * TILE_DBL, TILE_BYTES, &full[s]);
      if (++pt == P.nt) pt = ++pb * TPB;
    }
  }
  const double a = P.a, inv2a = 0.5 / P.a;
  const double hsc = 1.0;  // h, H unscaled: k1_group keeps 2a r.n (the 1/(2a) is folded into q~)

  double tg[R][TN], acc[R][3], hs[R][2];
  int slot[R];
  int loaded_b = -1, par = 0, h_m0 = -1, h_b = -1, fs = 0, nslot = 0;
  for (long long u = u0; u < u1; ++u) {
    const int i = (int)(u - u0);
    const int buf = i % NS;
    const unsigned parity = (unsigned)(i / NS) & 1u;
    if (b_cur != loaded_b) {
      if (loaded_b >= 0) {  // this CTA's target-side sums over block loaded_b: segment blockIdx.x + loaded_b
        double* sg = P.pseg + (size_t)(blockIdx.x + loaded_b) * KS_B * 3;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int tl = warp * 32 * R + r * 32 + lane;
          sg[3 * tl] = acc[r][0];
          sg[3 * tl + 1] = acc[r][1];
          sg[3 * tl + 2] = acc[r][2];
        }
      }
      loaded_b = b_cur;
      fs = min(b_cur * KS_B / P.nq, P.np - 1);  // target spheres of the block: fs .. fs + nslot - 1
      nslot = min((b_cur * KS_B + KS_B - 1) / P.nq, P.np - 1) - fs + 1;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int t = b_cur * KS_B + warp * 32 * R + r * 32 + lane;  // < npad
        const double* rec = P.pk + (size_t)REC * t;
#pragma unroll
        for (int c = 0; c < TN; ++c) {
          if (TQ && c >= 3) tqs[(c - 3) * KS_B + warp * 32 * R + r * 32 + lane] = rec[c];
          else tg[r][c] = rec[c];
        }
        slot[r] = min(t / P.nq, P.np - 1) - fs;
        acc[r][0] = acc[r][1] = acc[r][2] = 0.0;
      }
    }
    const int s0 = t_cur * K1_TS;
    const bool diag = t_cur < (b_cur + 1) * TPB;
    mbar_wait(&full[buf], parity);
    if (MODE != MODE_S && !diag) {  // H[slot][j] = (|y_j - c_slot|^2 - a^2)/(2a) for this tile,
      // each 32-source group stored twice in a row so that lane + k indexes it without a wrap
      for (int e = tid; e < nslot * K1_TS; e += blockDim.x) {
        const int sl = e / K1_TS, j = e - sl * K1_TS;
        const double* y = ring[buf] + j * REC;
        const double* c = cs + 3 * (fs + sl);
        const double d0 = y[0] - c[0], d1 = y[1] - c[1], d2 = y[2] - c[2];
        const double H = (fma(d2, d2, fma(d1, d1, d0 * d0)) - a * a) * hsc;
        double* row = Hs + sl * (2 * K1_TS) + (j >> 5) * 64 + (j & 31);
        row[0] = H;
        row[32] = H;
      }
      __syncthreads();
    }
#pragma unroll 1
    for (int grp = 0; grp < K1_TS / 32; ++grp) {
      // source spheres of this 32-point group (Nq >= 32: at most two): the first m0, the
      // second from in-tile index jb on; h per (target, source sphere) when m0 changes
      const int sg0 = s0 + 32 * grp;
      const int m0 = min(sg0 / P.nq, P.np - 1);
      const int m1 = min(m0 + 1, P.np - 1);
      const int jb = 32 * grp + (m0 + 1) * P.nq - sg0;
      if (MODE != MODE_S && (m0 != h_m0 || b_cur != h_b)) {
        h_m0 = m0;
        h_b = b_cur;
#pragma unroll
        for (int r = 0; r < R; ++r) {
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const double* c = cs + 3 * (q ? m1 : m0);
            const double d0 = tg[r][0] - c[0], d1 = tg[r][1] - c[1], d2 = tg[r][2] - c[2];
            hs[r][q] = (fma(d2, d2, fma(d1, d1, d0 * d0)) - a * a) * hsc;
          }
        }
      }
      const double* gr = ring[buf] + grp * 32 * REC;
      double as0 = 0.0, as1 = 0.0, as2 = 0.0;
      const bool mixed = jb < grp * 32 + 32;
      const double* tql = tqs + warp * 32 * R + lane;
      if (diag) {
        k1_group<MODE, R, false, true, UNR, TQ>(gr, tg, hs, grp * 32, jb, inv2a, Hs, slot, acc, lane, as0, as1, as2,
                                                tql, KS_B);
      } else {
        if (mixed)
          k1_group<MODE, R, true, true, UNR, TQ>(gr, tg, hs, grp * 32, jb, inv2a, Hs, slot, acc, lane, as0, as1,
                                                 as2, tql, KS_B);
        else
          k1_group<MODE, R, true, false, UNR, TQ>(gr, tg, hs, grp * 32, jb, inv2a, Hs, slot, acc, lane, as0, as1,
                                                  as2, tql, KS_B);
        double* rw = red[par][warp] + (grp * 32 + lane) * 3;
        rw[0] = as0;
        rw[1] = as1;
        rw[2] = as2;
      }
    }
    __syncthreads();  // ring[buf] consumed by every warp; red[par] complete
    if (!diag) {  // 192 values per tile: every thread of the block takes its share (4-warp shapes have 128)
      for (int e = tid; e < K1_TS * 3; e += 32 * KS_W) {
        double sum = 0.0;
#pragma unroll
        for (int w = 0; w < KS_W; ++w) sum += red[par][w][e];
        P.psrc[(size_t)b_cur * P.psrc_ld + 3 * (size_t)t_cur * K1_TS + e] = sum;
      }
      par ^= 1;
    }
    if (tid == 0 && u + NS < u1) {
      mbar_expect_tx(&full[buf], TILE_BYTES);
      bulk_g2s(ring[buf], P.pk + (size_t)pt * TILE_DBL, TILE_BYTES, &full[buf]);
      if (++pt == P.nt) pt = ++pb * TPB;
    }
    if (++t_cur == P.nt) t_cur = ++b_cur * TPB;
  }
  {
    double* sg = P.pseg + (size_t)(blockIdx.x + loaded_b) * KS_B * 3;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int tl = warp * 32 * R + r * 32 + lane;
      sg[3 * tl] = acc[r][0];
      sg[3 * tl + 1] = acc[r][1];
      sg[3 * tl + 2] = acc[r][2];
    }
  }
}

// ---------------------------------------------------------------- row reduction
// out[3 i + c] = (K1: the CTA segments over i's block in CTA order, then the source-side
// partials of blocks b' < b in block order -- or far[3 i + c]) + (K2: the near partials of
// row i in (target, source sphere) order).  A fixed summation order: the operator is
// bit-reproducible run to run (no floating-point atomics anywhere on the path).
struct RowRedParams {
  int N, r0, r1;
  const double *pseg, *psrc;  // K1 partials (pseg == nullptr: use far); psrc: symmetric kernel only
  size_t psrc_ld;
  int ks_b, tpb, nt, grid;
  int tri;                    // 1: symmetric kernel (block b has nt - b tpb units); 0: one-directional
  int t0;                     // one-directional: first target row of the launch (blocks from t0)
  long long ubeg, units;
  const double* far;
  const double* pinc;         // K2 partials [n_inc][3] (K2 order) or nullptr
  const int *row_ptr, *row_pos;
  double* out;
};

__device__ __forceinline__ int k1_cta_of(long long u, long long ubeg, long long units, int G) {
  int lo = 0, hi = G - 1;  // largest c with ubeg + units c / G <= u
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (ubeg + units * mid / G <= u) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__global__ void k_row_reduce(RowRedParams P) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x + 3LL * P.r0;
  if (e >= 3LL * P.r1) return;
  const int i = (int)(e / 3), c = (int)(e - 3LL * i);
  double v = 0.0;
  if (P.pseg) {
    const int il = i - P.t0;
    const int b = il / P.ks_b, local = il - b * P.ks_b;
    // units of block b: symmetric kernel nt - b tpb (tiles from the block's first on), else nt
    const long long Ub = P.tri ? (long long)b * P.nt - (long long)P.tpb * b * (b - 1) / 2 : (long long)b * P.nt;
    const long long nu = P.tri ? (P.nt - (long long)b * P.tpb) : (long long)P.nt;
    const long long lo = max(Ub, P.ubeg), hi = min(Ub + nu, P.ubeg + P.units);
    if (lo < hi) {
      const int c0 = k1_cta_of(lo, P.ubeg, P.units, P.grid), c1 = k1_cta_of(hi - 1, P.ubeg, P.units, P.grid);
      for (int cc = c0; cc <= c1; ++cc) v += P.pseg[((size_t)(cc + b) * P.ks_b + local) * 3 + c];
    }
    if (P.tri)
      for (int bb = 0; bb < b; ++bb) v += P.psrc[(size_t)bb * P.psrc_ld + e];
  } else if (P.far) {
    v = P.far[e];
  }
  if (P.pinc)
    for (int k = P.row_ptr[i]; k < P.row_ptr[i + 1]; ++k) v += P.pinc[3 * (size_t)P.row_pos[k] + c];
  P.out[e] = v;
}

void launch_row_reduce(Geom& g, bool k1_partials, const double* far, bool with_k2, double* out, int r0, int r1,
                       cudaStream_t st) {
  RowRedParams P{};
  P.N = g.n;
  P.r0 = r0;
  P.r1 = r1;
  if (k1_partials) {
    P.pseg = g.k1_pseg.p;
    P.psrc = g.k1_psrc.p;
    P.psrc_ld = g.k1lay.psrc_ld;
    P.ks_b = g.k1lay.ks_b;
    P.tpb = g.k1lay.tpb;
    P.nt = g.k1lay.nt;
    P.grid = g.k1lay.grid;
    P.tri = g.k1lay.sym ? 1 : 0;
    P.t0 = g.k1lay.t0;
    P.ubeg = g.k1lay.ubeg;
    P.units = g.k1lay.units;
  }
  P.far = far;
  P.pinc = with_k2 && g.n_inc > 0 ? g.k2_pinc.p : nullptr;
  P.row_ptr = g.row_ptr.p;
  P.row_pos = g.row_pos.p;
  P.out = out;
  const long long n = 3LL * (r1 - r0);
  if (n <= 0) return;
  k_row_reduce<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(P);
  BPQN_CHECK_LAUNCH();
  g.prof.launches++;
}

// Algorithmic flops per target-source pair of the fused formulation (DESIGN.md
// "Roofline"): S 28, D 29, S+D 42 (the rsqrt counted as one operation).
double allpairs_flops_per_pair(int mode) { return mode == MODE_S ? 28.0 : (mode == MODE_D ? 29.0 : 42.0); }

template <class K>
static int k1_grid(Geom& g, K kern, int threads) {
  int b = 0;
  BPQN_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, threads, 0));
  return std::max(1, b) * g.sms;
}

// K1 variant: symmetric (default) or one-directional (BPQN_K1=asym; A/B and self-check)
static bool k1_symmetric() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BPQN_K1");
    v = (e && std::string(e) == "asym") ? 0 : 1;
  }
  return v == 1;
}

template <int MODE, int W, int R, int MINB, int UNR = 2, bool TQ = false>
static void launch_sym_cfg(Geom& g, double* out, cudaStream_t st) {
  constexpr int KS_B = 32 * R * W;
  K1SymParams P;
  P.pk = g.packed.p;
  P.centers = g.centers_d.p;
  P.pseg = g.k1_pseg.p;
  P.psrc = g.k1_psrc.p;
  P.N = g.n;
  P.nq = g.nq;
  P.np = g.np;
  P.a = g.a;
  P.nb = (g.n + KS_B - 1) / KS_B;
  P.nt = P.nb * (KS_B / K1_TS);
  long long tot = 0;
  for (int b = 0; b < P.nb; ++b) tot += P.nt - b * (KS_B / K1_TS);
  // sharded symmetric K1: this rank's equal share of the unordered (block, tile) units
  P.ubeg = g.sharded() ? tot * g.shard_rank / g.shard_world : 0;
  P.units = g.sharded() ? tot * (g.shard_rank + 1) / g.shard_world - P.ubeg : tot;
  const int nslot_max = KS_B / g.nq + 2;
  const int smem = (K1_STAGES * K1_TS * RecS<MODE>::n + 2 * W * K1_TS * 3 + (TQ ? (TgtN<MODE>::n - 3) * KS_B : 0) +
                    (MODE == MODE_S ? 0 : 3 * g.np + nslot_max * 2 * K1_TS)) * 8;
  // per instantiation: the opt-in smem limit only grows; occupancy cached per smem size
  // (hi and lo fidelity handles alternate in Bi-PQN with different table sizes)
  static std::mutex mu;
  static int attr_smem = 0;
  static std::vector<std::pair<int, int>> occ;  // (smem, grid)
  int grid = 0;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (smem > attr_smem) {
      BPQN_CUDA(cudaFuncSetAttribute(k1_sym<MODE, W, R, MINB, UNR, TQ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     smem));
      attr_smem = smem;
    }
    for (auto& e : occ)
      if (e.first == smem) grid = e.second;
    if (!grid) {
      int b = 0;
      BPQN_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k1_sym<MODE, W, R, MINB, UNR, TQ>, 32 * W, smem));
      grid = std::max(1, b) * g.sms;
      occ.emplace_back(smem, grid);
    }
  }
  const int gr = (int)std::max<long long>(1, std::min<long long>(grid, P.units));
  const int npad = P.nb * KS_B;
  P.psrc_ld = 3 * (size_t)npad;
  K1Layout& Ly = g.k1lay;
  Ly.sym = true;
  Ly.ks_b = KS_B;
  Ly.tpb = KS_B / K1_TS;
  Ly.nt = P.nt;
  Ly.nb = P.nb;
  Ly.grid = gr;
  Ly.ubeg = P.ubeg;
  Ly.units = P.units;
  Ly.psrc_ld = P.psrc_ld;
  BPQN_REQUIRE((size_t)(gr + P.nb) * KS_B * 3 <= g.k1_pseg.n && (size_t)P.nb * P.psrc_ld <= g.k1_psrc.n,
               "K1 partial-sum workspace too small");
  if (g.sharded()) {  // this rank's share of the units: the other partials read as zero
    BPQN_CUDA(cudaMemsetAsync(g.k1_pseg.p, 0, sizeof(double) * (size_t)(gr + P.nb) * KS_B * 3, st));
    BPQN_CUDA(cudaMemsetAsync(g.k1_psrc.p, 0, sizeof(double) * (size_t)P.nb * P.psrc_ld, st));
  }
  if (P.units == 0) return;  // a rank with no share (more ranks than units): every partial stays zero
  k1_sym<MODE, W, R, MINB, UNR, TQ><<<gr, 32 * W, smem, st>>>(P);
}

static int sym_block_points(int c);
// Workspace of the symmetric kernel's partial sums for one launch shape.
static void sym_ws(const Geom& g, int cfg, size_t& pseg, size_t& psrc, size_t& packed) {
  const int kb = sym_block_points(cfg);
  const size_t nb = (size_t)((g.n + kb - 1) / kb), npad = nb * kb;
  pseg = std::max(pseg, (size_t)(4 * g.sms + nb) * kb * 3);  // grid <= 4 CTAs per SM
  psrc = std::max(psrc, nb * 3 * npad);
  packed = std::max(packed, npad * 14);
}

// Launch shape, measured on B200 (profiles/r01_k1_sym_shapes.md): 8 warps at 1 CTA/SM with
// 5 (D, S) or 4 (S+D) targets/lane for N >= 6e4 (c4: D 14.81, S 15.65, S+D 22.60 ms), 4 targets/lane
// for N >= 2e4 (c3 D 1.355 vs 1.46 ms with 3; c4 centres at p = 8: 1.14 vs 1.17 ms), 8 x 3 below, and
// 4 x 3 (two CTAs per SM) below N = 4000 (c1: 0.022 vs 0.028 ms; profiles/r02_k1_v8_ncu.md).
// BPQN_K1_CFG = 0..3 forces one shape for A/B runs.
static int k1_cfg() {
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("BPQN_K1_CFG");
    v = e ? atoi(e) : -1;
  }
  return v;
}

static int sym_cfg(const Geom& g, int mode) {
  const int c = k1_cfg();
  if (c >= 0) return c;
  return g.n >= 60000 ? (mode == MODE_SD ? 4 : 14) : (g.n >= 20000 ? 4 : (g.n >= 4000 ? 3 : 6));
}

// target-block size 32 W R of each launch shape (must match launch_sym's table): the packed
// records must cover nb blocks of it
static int sym_block_points(int c) {
  switch (c) {
    case 1: case 5: case 8: return 32 * 12 * 3;
    case 2: return 32 * 16 * 2;
    case 3: case 9: return 32 * 8 * 3;
    case 4: case 10: return 32 * 8 * 4;
    case 6: return 32 * 4 * 3;
    case 7: return 32 * 6 * 3;
    case 11: return 32 * 4 * 4;
    case 12: case 13: return 32 * 12 * 4;
    case 14: return 32 * 8 * 5;
    case 15: return 32 * 8 * 6;
    case 16: return 32 * 4 * 6;
    case 17: return 32 * 8 * 5;
    case 18: return 32 * 8 * 6;
    case 19: return 32 * 12 * 4;
    case 20: return 32 * 12 * 3;
    case 21: return 32 * 16 * 3;
    case 22: return 32 * 8 * 4;
    default: return 32 * 8 * 2;
  }
}

template <int MODE>
static void launch_sym(Geom& g, double* out, cudaStream_t st) {
  const int c = sym_cfg(g, MODE);
  switch (c) {
    case 1: launch_sym_cfg<MODE, 12, 3, 1>(g, out, st); break;
    case 2: launch_sym_cfg<MODE, 16, 2, 1>(g, out, st); break;
    case 3: launch_sym_cfg<MODE, 8, 3, 1>(g, out, st); break;
    case 4: launch_sym_cfg<MODE, 8, 4, 1>(g, out, st); break;
    case 5: launch_sym_cfg<MODE, 12, 3, 1, 1>(g, out, st); break;
    case 6: launch_sym_cfg<MODE, 4, 3, 3>(g, out, st); break;
    case 7: launch_sym_cfg<MODE, 6, 3, 2>(g, out, st); break;
    case 8: launch_sym_cfg<MODE, 12, 3, 1, 4>(g, out, st); break;
    case 9: launch_sym_cfg<MODE, 8, 3, 2>(g, out, st); break;
    case 10: launch_sym_cfg<MODE, 8, 4, 1, 1>(g, out, st); break;
    case 11: launch_sym_cfg<MODE, 4, 4, 2>(g, out, st); break;
    case 12: launch_sym_cfg<MODE, 12, 4, 1>(g, out, st); break;
    case 13: launch_sym_cfg<MODE, 12, 4, 1, 1>(g, out, st); break;
    case 14: launch_sym_cfg<MODE, 8, 5, 1>(g, out, st); break;
    case 15: launch_sym_cfg<MODE, 8, 6, 1>(g, out, st); break;
    case 16: launch_sym_cfg<MODE, 4, 6, 2>(g, out, st); break;
    case 17: launch_sym_cfg<MODE, 8, 5, 1, 2, true>(g, out, st); break;
    case 18: launch_sym_cfg<MODE, 8, 6, 1, 2, true>(g, out, st); break;
    case 19: launch_sym_cfg<MODE, 12, 4, 1, 2, true>(g, out, st); break;
    case 20: launch_sym_cfg<MODE, 12, 3, 1, 2, true>(g, out, st); break;
    case 21: launch_sym_cfg<MODE, 16, 3, 1, 2, true>(g, out, st); break;
    case 22: launch_sym_cfg<MODE, 8, 4, 1, 2, true>(g, out, st); break;
    default: launch_sym_cfg<MODE, 8, 2, 2>(g, out, st); break;
  }
}

template <int MODE>
static void launch_asym(Geom& g, double* out, cudaStream_t st, int t0, int t1) {
  K1Params P;
  P.t0 = t0;
  P.nt = t1 - t0;
  P.n_tb = (P.nt + K1_TB - 1) / K1_TB;
  P.n_st = (g.n + K1_TS - 1) / K1_TS;
  P.units = (long long)P.n_tb * P.n_st;
  P.X = g.X.p;
  P.pk = g.packed.p;
  P.pseg = g.k1_pseg.p;
  static int grid = 0;
  if (!grid) grid = k1_grid(g, k1_allpairs<MODE>, K1_THREADS);
  const int gr = (int)std::max<long long>(1, std::min<long long>(grid, P.units));
  K1Layout& Ly = g.k1lay;
  Ly.sym = false;
  Ly.ks_b = K1_TB;
  Ly.tpb = 0;
  Ly.nt = P.n_st;
  Ly.nb = P.n_tb;
  Ly.grid = gr;
  Ly.t0 = t0;
  Ly.ubeg = 0;
  Ly.units = P.units;
  Ly.psrc_ld = 0;
  BPQN_REQUIRE((size_t)(gr + P.n_tb) * K1_TB * 3 <= g.k1_pseg.n, "K1 partial-sum workspace too small");
  if (P.units == 0) return;
  k1_allpairs<MODE><<<gr, K1_THREADS, 0, st>>>(P);
}

// the symmetric kernel needs tiles that span <= 2 spheres and the centres in shared memory
static bool k1_sym_eligible(const Geom& g) { return g.nq >= 32 && g.np <= 4096; }

// Sharded handle whose K1 runs the symmetric kernel over this rank's share of the units: the
// partial sums cover every target row and must be reduce-scattered (layer.cu).
bool k1_sharded_symmetric(const Geom& g) {
  return g.sharded() && (g.sh_rs_fn != nullptr || g.sh_sym_nccl) && k1_symmetric() && k1_sym_eligible(g);
}

// All K1 workspace, allocated once per handle (geometry init / update): the packed records and
// the deterministic partial-sum buffers for every mode's launch shape -- the hot calls allocate nothing.
void k1_reserve(Geom& g) {
  // one-directional kernel: (grid + target blocks) segments of K1_TB rows (grid <= 4 CTAs per SM)
  size_t pseg = (size_t)(4 * g.sms + (g.n + K1_TB - 1) / K1_TB) * K1_TB * 3, psrc = 1,
         packed = ((g.n + K1_TS - 1) / K1_TS) * (size_t)K1_TS * 14;
  if (k1_sym_eligible(g))
    for (int mode = 0; mode < 3; ++mode) sym_ws(g, sym_cfg(g, mode), pseg, psrc, packed);
  g.k1_pseg.ensure(pseg);
  g.k1_psrc.ensure(psrc);
  g.packed.ensure(packed);
}

void launch_allpairs(Geom& g, int mode, const double* sigS, const double* sigD, double* out, cudaStream_t st) {
  const bool sym = k1_symmetric();
  // symmetric kernel: a 32-point group spans <= 2 spheres, centres fit smem, all targets on this
  // GPU (or the sharded symmetric split with its reduce-scatter)
  const bool use_sym = sym && k1_sym_eligible(g) && (!g.sharded() || g.sh_rs_fn != nullptr || g.sh_sym_nccl);
  // packed records cover every target block (symmetric: nb blocks of the launch shape) and
  // source tile (one-directional: 64-point tiles); the padding is far away, zero strength
  const int blk = use_sym ? sym_block_points(sym_cfg(g, mode)) : K1_TS;
  const int npad = ((g.n + blk - 1) / blk) * blk;
  BPQN_REQUIRE((size_t)npad * 14 <= g.packed.n, "K1 packed workspace too small (k1_reserve)");
  if (use_sym)
    k1_pack_sym<<<(npad + 255) / 256, 256, 0, st>>>(mode, g.n, npad, g.src.p, sigS, sigD,
                                                   1.0 / (8.0 * PI_A * g.mu),
                                                   // D mode: 1/(2a) folded into q~ (k1_group's 2a r.n)
                                                   -3.0 / (4.0 * PI_A) / (mode == MODE_S ? 1.0 : 2.0 * g.a),
                                                   g.packed.p);
  else
    k1_pack<<<(npad + 255) / 256, 256, 0, st>>>(mode, g.n, npad, g.src.p, sigS, sigD, 1.0 / (8.0 * PI_A * g.mu),
                                               -3.0 / (4.0 * PI_A), g.packed.p);
  BPQN_CHECK_LAUNCH();
  g.k1lay.sym = use_sym;
  g.k1lay.t0 = 0;
  if (use_sym) {
    if (mode == MODE_D) launch_sym<MODE_D>(g, out, st);
    else if (mode == MODE_S) launch_sym<MODE_S>(g, out, st);
    else launch_sym<MODE_SD>(g, out, st);
  } else {
    // sharded (bpqn_geometry_shard): this rank's target rows against all sources
    const int t0 = g.sharded() ? g.sh_t0 : 0, t1 = g.sharded() ? g.sh_t1 : g.n;
    if (mode == MODE_D) launch_asym<MODE_D>(g, out, st, t0, t1);
    else if (mode == MODE_S) launch_asym<MODE_S>(g, out, st, t0, t1);
    else launch_asym<MODE_SD>(g, out, st, t0, t1);
  }
  BPQN_CHECK_LAUNCH();
  g.prof.allpairs_launches++;
  g.prof.launches += 2;
}

}  // namespace bpqn
