// K5: contact detection and the small per-sphere maps around the mobility solve.
//  * contacts: Phi_l = |c_j - c_i| - 2a < delta over all pairs i < j (P:152-157,
//    R20), order-preserving compaction (lexicographic), normals n = (c_j-c_i)/|.|
//  * D lambda: F_i -= lambda_l n_l, F_j += lambda_l n_l, torques 0
//  * P^T (R2): f = F/(4 pi a^2) + 3/(8 pi a^3) T x xi
//  * rigid read-out (R4): (U, Omega) = -(Ubar[q], Obar[q])
//  * D^T: w_l = n_l . (U_j - U_i)
//  * Janus slip (R13)
// All launch-latency bound (Np <= 216, Nc <= 540).
#include <algorithm>
#include <cmath>

#include "bpqn_internal.h"

namespace bpqn {

static const double PI_C = 3.14159265358979323846;

// One CTA scans all Np(Np-1)/2 pairs in lexicographic order (chunks of blockDim),
// block-scans the flags and writes the compacted list.
__global__ void k_contacts(int np, const double* c, double a, double thr, int cap, int* pairs, double* normals,
                           double* gaps, int* count) {
  __shared__ int warp_sums[32];
  __shared__ int base;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  const long long npairs = (long long)np * (np - 1) / 2;
  for (long long p0 = 0; p0 < npairs; p0 += blockDim.x) {
    long long pid = p0 + threadIdx.x;
    int flag = 0, i = 0, j = 0;
    double gap = 0, nx = 0, ny = 0, nz = 0;
    if (pid < npairs) {
      // invert pid -> (i, j), i < j, lexicographic
      long long rem = pid;
      i = 0;
      while (rem >= np - 1 - i) {
        rem -= np - 1 - i;
        ++i;
      }
      j = i + 1 + (int)rem;
      double dx = c[3 * j] - c[3 * i], dy = c[3 * j + 1] - c[3 * i + 1], dz = c[3 * j + 2] - c[3 * i + 2];
      double d = sqrt(dx * dx + dy * dy + dz * dz);
      gap = d - 2.0 * a;
      flag = gap < thr;
      nx = dx / d; ny = dy / d; nz = dz / d;
    }
    // block exclusive scan of flag
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int v = flag;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += t;
    }
    if (lane == 31) warp_sums[wid] = v;
    __syncthreads();
    if (wid == 0) {
      int nw = blockDim.x >> 5;
      int s = lane < nw ? warp_sums[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += t;
      }
      if (lane < nw) warp_sums[lane] = s;
    }
    __syncthreads();
    int incl = v + (wid > 0 ? warp_sums[wid - 1] : 0);
    int pos = base + incl - flag;
    if (flag && pos < cap) {
      pairs[2 * pos] = i;
      pairs[2 * pos + 1] = j;
      normals[3 * pos] = nx; normals[3 * pos + 1] = ny; normals[3 * pos + 2] = nz;
      gaps[pos] = gap;
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) base += incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) *count = base;
}

int detect_contacts(Geom& g, double thr, int max_contacts, int* pairs, double* normals, double* gaps,
                    cudaStream_t st) {
  DBuf<int> cnt;
  cnt.alloc(1);
  k_contacts<<<1, 1024, 0, st>>>(g.np, g.centers_d.p, g.a, thr, max_contacts, pairs, normals, gaps, cnt.p);
  BPQN_CHECK_LAUNCH();
  int h = 0;
  BPQN_CUDA(cudaMemcpyAsync(&h, cnt.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  BPQN_CUDA(cudaStreamSynchronize(st));
  return h;
}

// ft[m] = sum over contacts touching m of -+ lambda n (one thread per sphere, deterministic order)
__global__ void k_d_scatter(int np, int nc, const int* pairs, const double* normals, const double* lam, double* ft) {
  int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= np) return;
  double f0 = 0, f1 = 0, f2 = 0;
  for (int l = 0; l < nc; ++l) {
    int i = pairs[2 * l], j = pairs[2 * l + 1];
    double s = (m == i) ? -lam[l] : ((m == j) ? lam[l] : 0.0);
    if (s != 0.0) {
      f0 = fma(s, normals[3 * l], f0);
      f1 = fma(s, normals[3 * l + 1], f1);
      f2 = fma(s, normals[3 * l + 2], f2);
    }
  }
  ft[6 * m] = f0; ft[6 * m + 1] = f1; ft[6 * m + 2] = f2;
  ft[6 * m + 3] = 0.0; ft[6 * m + 4] = 0.0; ft[6 * m + 5] = 0.0;
}

void launch_d_scatter(Geom& g, const double* lam, double* ft, cudaStream_t st) {
  k_d_scatter<<<(g.np + 127) / 128, 128, 0, st>>>(g.np, g.nc, g.pairs.p, g.normals.p, lam, ft);
  BPQN_CHECK_LAUNCH();
  g.prof.launches++;
}

__global__ void k_pt(int n, int nq, double a, const double* xi, const double* ft, double* f) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int m = i / nq, k = i - m * nq;
  const double* F = ft + 6 * m;
  double x0 = xi[3 * k], x1 = xi[3 * k + 1], x2 = xi[3 * k + 2];
  double cf = 1.0 / (4.0 * PI_C * a * a), ct = 3.0 / (8.0 * PI_C * a * a * a);
  f[3 * i] = cf * F[0] + ct * (F[4] * x2 - F[5] * x1);
  f[3 * i + 1] = cf * F[1] + ct * (F[5] * x0 - F[3] * x2);
  f[3 * i + 2] = cf * F[2] + ct * (F[3] * x1 - F[4] * x0);
}

void launch_pt(Geom& g, const double* ft, double* f, cudaStream_t st) {
  k_pt<<<(g.n + 255) / 256, 256, 0, st>>>(g.n, g.nq, g.a, g.xi_d.p, ft, f);
  BPQN_CHECK_LAUNCH();
  g.prof.launches++;
}

// one CTA per sphere: uo = -(sum w q / (4 pi a^2), 3/(8 pi a^4) sum w (x-c) x q)
__global__ void k_rigid(int nq, double a, const double* xi, const double* w, const double* q, double* uo) {
  const int m = blockIdx.x;
  double acc[6] = {0, 0, 0, 0, 0, 0};
  for (int k = threadIdx.x; k < nq; k += blockDim.x) {
    const double* qq = q + 3 * ((size_t)m * nq + k);
    double wk = w[k];
    double r0 = a * xi[3 * k], r1 = a * xi[3 * k + 1], r2 = a * xi[3 * k + 2];
    acc[0] += wk * qq[0];
    acc[1] += wk * qq[1];
    acc[2] += wk * qq[2];
    acc[3] += wk * (r1 * qq[2] - r2 * qq[1]);
    acc[4] += wk * (r2 * qq[0] - r0 * qq[2]);
    acc[5] += wk * (r0 * qq[1] - r1 * qq[0]);
  }
  __shared__ double sred[6][32];
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    double v = acc[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) sred[c][wid] = v;
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    double s = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s += sred[threadIdx.x][k];
    double scale = threadIdx.x < 3 ? 1.0 / (4.0 * PI_C * a * a) : 3.0 / (8.0 * PI_C * a * a * a * a);
    uo[6 * m + threadIdx.x] = -scale * s;
  }
}

void launch_rigid_readout(Geom& g, const double* q, double* uo, cudaStream_t st) {
  k_rigid<<<g.np, 256, 0, st>>>(g.nq, g.a, g.xi_d.p, g.w_d.p, q, uo);
  BPQN_CHECK_LAUNCH();
  g.prof.launches++;
}

// w_l = scale * n_l . (U_j - U_i) (+ add_l)
__global__ void k_dt(int nc, const int* pairs, const double* normals, const double* uo, double scale,
                     const double* add, double* w) {
  int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= nc) return;
  int i = pairs[2 * l], j = pairs[2 * l + 1];
  double v = normals[3 * l] * (uo[6 * j] - uo[6 * i]) + normals[3 * l + 1] * (uo[6 * j + 1] - uo[6 * i + 1]) +
             normals[3 * l + 2] * (uo[6 * j + 2] - uo[6 * i + 2]);
  v *= scale;
  if (add) v += add[l];
  w[l] = v;
}

void launch_dt_gather(Geom& g, const double* uo, double* w, double scale, const double* add, cudaStream_t st) {
  if (g.nc == 0) return;
  k_dt<<<(g.nc + 127) / 128, 128, 0, st>>>(g.nc, g.pairs.p, g.normals.p, uo, scale, add, w);
  BPQN_CHECK_LAUNCH();
  g.prof.launches++;
}

__global__ void k_axpby(double* y, double a, const double* x, double b, size_t n) {
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x)
    y[e] = a * x[e] + b * y[e];
}

void launch_axpby(double* y, double a, const double* x, double b, size_t n, cudaStream_t st) {
  int blocks = (int)std::min<size_t>((n + 255) / 256, 148 * 8);
  k_axpby<<<blocks, 256, 0, st>>>(y, a, x, b, n);
  BPQN_CHECK_LAUNCH();
}

__global__ void k_slip(int n, int nq, const double* xi, const double* axes, double B, double* us) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int m = i / nq, k = i - m * nq;
  double a0 = axes[3 * m], a1 = axes[3 * m + 1], a2 = axes[3 * m + 2];
  double x0 = xi[3 * k], x1 = xi[3 * k + 1], x2 = xi[3 * k + 2];
  double c = x0 * a0 + x1 * a1 + x2 * a2;
  if (c > 0.0) {
    us[3 * i] = -B * (a0 - c * x0);
    us[3 * i + 1] = -B * (a1 - c * x1);
    us[3 * i + 2] = -B * (a2 - c * x2);
  } else {
    us[3 * i] = us[3 * i + 1] = us[3 * i + 2] = 0.0;
  }
}

void launch_slip(Geom& g, const double* axes_dev, double B, double* slip, cudaStream_t st) {
  k_slip<<<(g.n + 255) / 256, 256, 0, st>>>(g.n, g.nq, g.xi_d.p, axes_dev, B, slip);
  BPQN_CHECK_LAUNCH();
}

}  // namespace bpqn
