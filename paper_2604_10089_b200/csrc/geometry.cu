// P0: geometry precompute for libbpqn (B200 / sm_100a).
//
// Builds, for one discretisation (readings R5-R8, R10):
//  * the order-p grid (Gauss-Legendre in cos(theta) x trapezoid in phi),
//  * the SH analysis matrix of the projection onto V_p (R7: quadrature analysis
//    with the cos(p phi) sectoral coefficient halved, App. A.3 of SURVEY),
//  * the per-sphere self operators E_S, E_L, E_A  (rotated singular grid, R5/R6;
//    computed for one target per polar ring and expanded by the exact z-rotation
//    symmetry of the grid),
//  * the near-incidence refined tensors T_S, T_D (sinh-graded polar rule, R8) in
//    SH-coefficient space, one [6][nb] block per (target, sphere); K2 applies them to
//    the density's SH coefficients and subtracts the coarse rule on the fly.
// The paper names none of this (PAPER.md P:425-426 only gives the dof count and
// cost); it is the discretisation frozen in DESIGN.md, implemented independently
// of the CPU oracle.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

#include "bpqn_internal.h"

namespace bpqn {

static const double PI = 3.14159265358979323846;

// ------------------------------------------------------------------ host grids
// Gauss-Legendre nodes by Newton iteration on P_n (own implementation), DESCENDING.
void gauss_legendre_desc(int n, std::vector<double>& t, std::vector<double>& w) {
  t.assign(n, 0.0);
  w.assign(n, 0.0);
  for (int i = 0; i < n; ++i) {
    double x = std::cos(PI * (i + 0.75) / (n + 0.5));
    double dp = 0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = x;
      for (int k = 2; k <= n; ++k) {
        double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      double pn = (n == 0) ? 1.0 : (n == 1 ? x : p1);
      double pm1 = (n == 1) ? 1.0 : p0;
      dp = n * (x * pn - pm1) / (x * x - 1.0);
      double dx = pn / dp;
      x -= dx;
      if (std::fabs(dx) < 1e-16) {
        // one more evaluation for the derivative at the converged node
        p0 = 1.0;
        p1 = x;
        for (int k = 2; k <= n; ++k) {
          double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
          p0 = p1;
          p1 = p2;
        }
        pn = (n == 1) ? x : p1;
        pm1 = (n == 1) ? 1.0 : p0;
        dp = n * (x * pn - pm1) / (x * x - 1.0);
        break;
      }
    }
    t[i] = x;
    w[i] = 2.0 / ((1.0 - x * x) * dp * dp);
  }
  // symmetrise (nodes come in +- pairs)
  for (int i = 0; i < n / 2; ++i) {
    double tt = 0.5 * (t[i] - t[n - 1 - i]);
    double ww = 0.5 * (w[i] + w[n - 1 - i]);
    t[i] = tt;
    t[n - 1 - i] = -tt;
    w[i] = w[n - 1 - i] = ww;
  }
  if (n % 2) t[n / 2] = 0.0;
}

void build_grid(int p, double a, Grid& g) {
  g.p = p;
  g.nq = (p + 1) * 2 * p;
  gauss_legendre_desc(p + 1, g.t, g.omega);
  g.theta.resize(p + 1);
  for (int k = 0; k <= p; ++k) g.theta[k] = std::acos(g.t[k]);
  g.phi.resize(2 * p);
  for (int l = 0; l < 2 * p; ++l) g.phi[l] = PI * l / p;
  g.xi.resize(3 * g.nq);
  g.w.resize(g.nq);
  for (int k = 0; k <= p; ++k)
    for (int l = 0; l < 2 * p; ++l) {
      int i = k * 2 * p + l;
      double st = std::sqrt(std::max(0.0, 1.0 - g.t[k] * g.t[k]));
      g.xi[3 * i] = st * std::cos(g.phi[l]);
      g.xi[3 * i + 1] = st * std::sin(g.phi[l]);
      g.xi[3 * i + 2] = g.t[k];
      g.w[i] = a * a * g.omega[k] * PI / p;
    }
}

int sh_count(int p) { return p * p + 2 * p; }

// ------------------------------------------------------------------ device SH
// Real orthonormal SH of V_p at a unit vector eta, one m-column at a time:
//   Y^c_lm = sqrt(2 - d_m0) c_m Re[(x + i y)^m] R_lm(z),  Y^s_lm = sqrt2 c_m Im[...] R_lm(z)
// with c_m = Q_mm / sin^m (Q normalised on the sphere) and R_lm = Q_lm/Q_mm by the
// three-term recurrence.  Basis index: cos-type m = 0..p, l = m..p first
// (offset m(p+1) - m(m-1)/2), then sin-type m = 1..p-1, l = m..p (sin p phi dropped).
struct ShTables {
  const double* ra;  // [(p+1)*(p+1)] recurrence a_lm at l*(p+1)+m
  const double* rb;  // b_lm
  const double* cm;  // [p+1]
};

__host__ __device__ inline int sh_cos_index(int p, int l, int m) { return m * (p + 1) - m * (m - 1) / 2 + (l - m); }
__host__ __device__ inline int sh_sin_index(int p, int l, int m) {
  int nc = (p + 1) * (p + 2) / 2;
  int mm = m - 1;  // m >= 1
  return nc + mm * p - mm * (mm - 1) / 2 + (l - m);
}

// writes Y for column m into out[idx*stride]
__device__ void sh_column(int p, int m, double ex, double ey, double ez, const ShTables& T, double* out,
                          int stride) {
  // (x + i y)^m
  double re = 1.0, im = 0.0;
  for (int k = 0; k < m; ++k) {
    double nr = re * ex - im * ey;
    im = re * ey + im * ex;
    re = nr;
  }
  const double s2 = 1.4142135623730951;
  double cc = (m == 0) ? T.cm[0] : s2 * T.cm[m] * re;
  double ss = s2 * T.cm[m] * im;
  double rm2 = 0.0, rm1 = 0.0;
  for (int l = m; l <= p; ++l) {
    double r;
    if (l == m) r = 1.0;
    else if (l == m + 1) r = T.ra[l * (p + 1) + m] * ez;
    else r = T.ra[l * (p + 1) + m] * (ez * rm1 - T.rb[l * (p + 1) + m] * rm2);
    rm2 = rm1;
    rm1 = r;
    out[(size_t)sh_cos_index(p, l, m) * stride] = cc * r;
    if (m >= 1 && m < p) out[(size_t)sh_sin_index(p, l, m) * stride] = ss * r;
  }
}

static void sh_tables_host(int p, std::vector<double>& ra, std::vector<double>& rb, std::vector<double>& cm) {
  ra.assign((p + 1) * (p + 1), 0.0);
  rb.assign((p + 1) * (p + 1), 0.0);
  cm.assign(p + 1, 0.0);
  cm[0] = 1.0 / std::sqrt(4.0 * PI);
  for (int m = 1; m <= p; ++m) cm[m] = cm[m - 1] * std::sqrt((2.0 * m + 1.0) / (2.0 * m));
  for (int m = 0; m <= p; ++m)
    for (int l = m + 1; l <= p; ++l) {
      if (l == m + 1) {
        ra[l * (p + 1) + m] = std::sqrt(2.0 * m + 3.0);
      } else {
        ra[l * (p + 1) + m] = std::sqrt((4.0 * l * l - 1.0) / ((double)l * l - (double)m * m));
        rb[l * (p + 1) + m] =
            std::sqrt(((l - 1.0) * (l - 1.0) - (double)m * m) / (4.0 * (l - 1.0) * (l - 1.0) - 1.0));
      }
    }
}

// analysis[b][j] = Y_b(xi_j) * omega_unit_j / G_bb (G = 2 for the cos(p phi) sectoral)
__global__ void k_analysis(int p, int nq, const double* xi, const double* wunit, ShTables T, double* Yn,
                           double* A, int nb) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nq) return;
  double ex = xi[3 * j], ey = xi[3 * j + 1], ez = xi[3 * j + 2];
  for (int m = 0; m <= p; ++m) sh_column(p, m, ex, ey, ez, T, Yn + j, nq);
  int bnyq = sh_cos_index(p, p, p);
  for (int b = 0; b < nb; ++b) A[(size_t)b * nq + j] = Yn[(size_t)b * nq + j] * wunit[j] * (b == bnyq ? 0.5 : 1.0);
}

// ------------------------------------------------------------------ quadrature -> rows
// One CTA per quadrature problem.  kind 0: self rule for polar ring k (target at
// (theta_k, phi = 0) on a sphere at the origin); kind 1: near rule for incidence
// (target x_i, source sphere m).  Produces, for every source node j of the sphere,
//   rowS[a][3j+c] = sum_s w_s G(x - y_s)[a][c]  Pi_j(eta_s)
//   rowD[a][3j+c] = sum_s w_s K_D(x, y_s)[a][c] Pi_j(eta_s)
// minus (kind 1) the coarse-rule terms w_j K(x - y_j) that the all-pairs kernel adds.
struct QuadParams {
  int p, nq, nb, kind;
  double a, mu;
  // self rule
  int ns_t, ns_p;          // theta' nodes (p_s+1), phi' nodes (2 p_s)
  const double* gl_self_t; // GL nodes on [-1,1] for theta' (p_s+1)
  const double* gl_self_w;
  const double* theta_ring;// [p+1]
  // near rule
  int n1, n2, nphi;
  double theta_c;
  const double* gl1_t; const double* gl1_w;
  const double* gl2_t; const double* gl2_w;
  const int* inc_t; const int* inc_m;
  const double* X;         // [N][3]
  const double* centers;   // [np][3]
  // common
  const double* xi;        // [nq][3]
  const double* w;         // [nq]
  const double* A;         // [nb][nq]
  ShTables T;
  double* outS;            // self rings: [nprob][3][3nq]; near incidences: [nprob][6][nb'] (K2 tensors)
  double* outD;
  int want_s;
};

constexpr int QT = 256;      // threads
constexpr int QPC = 16;      // points per chunk

__device__ inline void rot_apply(const double R[9], double x, double y, double z, double& ox, double& oy,
                                 double& oz) {
  ox = R[0] * x + R[1] * y + R[2] * z;
  oy = R[3] * x + R[4] * y + R[5] * z;
  oz = R[6] * x + R[7] * y + R[8] * z;
}

__global__ void __launch_bounds__(QT) k_quad_rows(QuadParams P) {
  extern __shared__ double sm[];
  const int prob = blockIdx.x;
  const int nb = P.nb, nq = P.nq, p = P.p;
  // smem layout
  double* sth = sm;                      // sin theta'     [ntheta <= 128]
  double* cth = sth + 128;               // cos theta'
  double* thw = cth + 128;               // theta' weights (incl. sin, a^2, dphi)
  double* cph = thw + 128;               // cos phi'       [nphi <= 256]
  double* sph = cph + 256;
  double* Kc = sph + 256;                // [QPC][12]
  double* Ys = Kc + QPC * 12;            // [QPC][nb]
  double* Tm = Ys + QPC * nb;            // [12][nb]
  __shared__ double R[9], tx[3], tc[3];
  __shared__ int ntheta, nphi;

  if (threadIdx.x == 0) {
    double ex, ey, ez, cx = 0, cy = 0, cz = 0, x0, x1, x2;
    if (P.kind == 0) {
      double t = P.theta_ring[prob];
      double c = cos(t), s = sin(t);
      // R = R_y(theta_k)
      R[0] = c; R[1] = 0; R[2] = s; R[3] = 0; R[4] = 1; R[5] = 0; R[6] = -s; R[7] = 0; R[8] = c;
      x0 = P.a * s; x1 = 0; x2 = P.a * c;
      ntheta = P.ns_t;
      nphi = P.ns_p;
    } else {
      int i = P.inc_t[prob], m = P.inc_m[prob];
      x0 = P.X[3 * i]; x1 = P.X[3 * i + 1]; x2 = P.X[3 * i + 2];
      cx = P.centers[3 * m]; cy = P.centers[3 * m + 1]; cz = P.centers[3 * m + 2];
      double rx = x0 - cx, ry = x1 - cy, rz = x2 - cz;
      double d = sqrt(rx * rx + ry * ry + rz * rz);
      ex = rx / d; ey = ry / d; ez = rz / d;
      double te = acos(fmin(1.0, fmax(-1.0, ez)));
      double pe = atan2(ey, ex);
      double ct = cos(te), st = sin(te), cp = cos(pe), sp = sin(pe);
      // R = R_z(pe) R_y(te)
      R[0] = cp * ct; R[1] = -sp; R[2] = cp * st;
      R[3] = sp * ct; R[4] = cp;  R[5] = sp * st;
      R[6] = -st;     R[7] = 0;   R[8] = ct;
      ntheta = P.n1 + P.n2;
      nphi = P.nphi;
    }
    tx[0] = x0; tx[1] = x1; tx[2] = x2;
    tc[0] = cx; tc[1] = cy; tc[2] = cz;
  }
  __syncthreads();
  const int nth = ntheta, nph = nphi;
  // theta' nodes and weights, phi' trig
  for (int k = threadIdx.x; k < nth; k += QT) {
    double tt, ww;
    if (P.kind == 0) {
      double t = P.gl_self_t[k], w = P.gl_self_w[k];
      tt = 0.5 * PI * (t + 1.0);
      ww = 0.5 * PI * w;
    } else {
      double rx = tx[0] - tc[0], ry = tx[1] - tc[1], rz = tx[2] - tc[2];
      double delta = (sqrt(rx * rx + ry * ry + rz * rz) - P.a) / P.a;
      if (k < P.n1) {
        double S = asinh(P.theta_c / delta);
        double s = 0.5 * S * (P.gl1_t[k] + 1.0);
        tt = delta * sinh(s);
        ww = 0.5 * S * P.gl1_w[k] * delta * cosh(s);
      } else {
        int kk = k - P.n1;
        tt = P.theta_c + 0.5 * (PI - P.theta_c) * (P.gl2_t[kk] + 1.0);
        ww = 0.5 * (PI - P.theta_c) * P.gl2_w[kk];
      }
    }
    sth[k] = sin(tt);
    cth[k] = cos(tt);
    thw[k] = ww * sth[k] * P.a * P.a * (2.0 * PI / nph);
  }
  for (int l = threadIdx.x; l < nph; l += QT) {
    double ph = 2.0 * PI * l / nph;
    cph[l] = cos(ph);
    sph[l] = sin(ph);
  }
  __syncthreads();

  // accumulator tiles: 3 kk-blocks (4 each) x nb/2 b-blocks
  const int nbb = (nb + 1) / 2;
  const int ntile = 3 * nbb;
  constexpr int MAXT = 4;  // tiles per thread: 3 ceil(nb/2) <= QT MAXT, i.e. p <= BPQN_P_MAX (checked on host)
  double acc[MAXT][8];
#pragma unroll
  for (int u = 0; u < MAXT; ++u)
#pragma unroll
    for (int v = 0; v < 8; ++v) acc[u][v] = 0.0;

  const double cS = 1.0 / (8.0 * PI * P.mu);
  const double cD = -3.0 / (4.0 * PI);
  const int npts = nth * nph;
  for (int s0 = 0; s0 < npts; s0 += QPC) {
    // phase A1: points and kernels
    for (int s = threadIdx.x; s < QPC; s += QT) {
      int sg = s0 + s;
      double k12[12];
      double ex = 0, ey = 0, ez = 1;
      if (sg < npts) {
        int it = sg / nph, ip = sg - it * nph;
        double st = sth[it], ct = cth[it];
        rot_apply(R, st * cph[ip], st * sph[ip], ct, ex, ey, ez);
        double wq = thw[it];
        double r0 = tx[0] - (tc[0] + P.a * ex), r1 = tx[1] - (tc[1] + P.a * ey), r2 = tx[2] - (tc[2] + P.a * ez);
        double rr = r0 * r0 + r1 * r1 + r2 * r2;
        double ir = 1.0 / sqrt(rr), ir2 = ir * ir, ir3 = ir * ir2;
        double gs = cS * wq;
        // G: (I/rho + r r^T/rho^3) ; order xx,xy,xz,yy,yz,zz
        k12[0] = gs * (ir + r0 * r0 * ir3); k12[1] = gs * r0 * r1 * ir3; k12[2] = gs * r0 * r2 * ir3;
        k12[3] = gs * (ir + r1 * r1 * ir3); k12[4] = gs * r1 * r2 * ir3; k12[5] = gs * (ir + r2 * r2 * ir3);
        double rn = r0 * ex + r1 * ey + r2 * ez;
        double kd = cD * wq * rn * ir3 * ir2;
        k12[6] = kd * r0 * r0; k12[7] = kd * r0 * r1; k12[8] = kd * r0 * r2;
        k12[9] = kd * r1 * r1; k12[10] = kd * r1 * r2; k12[11] = kd * r2 * r2;
      } else {
        for (int q = 0; q < 12; ++q) k12[q] = 0.0;
      }
      for (int q = 0; q < 12; ++q) Kc[s * 12 + q] = k12[q];
      // stash unit point in Ys row tail-free scratch: recompute in A2 instead
    }
    // phase A2: SH columns, work item = (s, m)
    for (int wi = threadIdx.x; wi < QPC * (p + 1); wi += QT) {
      int s = wi / (p + 1), m = wi - s * (p + 1);
      int sg = s0 + s;
      double ex = 0, ey = 0, ez = 1;
      if (sg < npts) {
        int it = sg / nph, ip = sg - it * nph;
        double st = sth[it], ct = cth[it];
        rot_apply(R, st * cph[ip], st * sph[ip], ct, ex, ey, ez);
      }
      sh_column(p, m, ex, ey, ez, P.T, Ys + s * nb, 1);
    }
    __syncthreads();
    // phase B: acc += Kc^T Ys over this chunk
#pragma unroll
    for (int u = 0; u < MAXT; ++u) {
      int tile = threadIdx.x + u * QT;
      if (tile < ntile) {
        int kb = tile / nbb, bb = tile - kb * nbb;
        int b0 = 2 * bb;
        bool two = (b0 + 1) < nb;
        for (int s = 0; s < QPC; ++s) {
          double y0 = Ys[s * nb + b0];
          double y1 = two ? Ys[s * nb + b0 + 1] : 0.0;
          const double* kr = Kc + s * 12 + 4 * kb;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            acc[u][2 * q] = fma(kr[q], y0, acc[u][2 * q]);
            acc[u][2 * q + 1] = fma(kr[q], y1, acc[u][2 * q + 1]);
          }
        }
      }
    }
    __syncthreads();
  }
  // write T [12][nb]
#pragma unroll
  for (int u = 0; u < MAXT; ++u) {
    int tile = threadIdx.x + u * QT;
    if (tile < ntile) {
      int kb = tile / nbb, bb = tile - kb * nbb;
      int b0 = 2 * bb;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        Tm[(4 * kb + q) * nb + b0] = acc[u][2 * q];
        if (b0 + 1 < nb) Tm[(4 * kb + q) * nb + b0 + 1] = acc[u][2 * q + 1];
      }
    }
  }
  __syncthreads();
  if (P.kind == 1) {  // near incidence: the refined tensors in SH-coefficient space (K2 applies them),
    // rows padded to an even length nbp (16-byte loads in K2) with zeros
    const int nbp = (nb + 1) & ~1;
    const size_t o = (size_t)prob * 6 * nbp;
    for (int e = threadIdx.x; e < 6 * nbp; e += QT) {
      const int q = e / nbp, b = e - q * nbp;
      P.outD[o + e] = b < nb ? Tm[(6 + q) * nb + b] : 0.0;
      if (P.want_s) P.outS[o + e] = b < nb ? Tm[q * nb + b] : 0.0;
    }
    return;
  }
  // phase C (self rings): rows over source nodes j
  const int sym[9] = {0, 1, 2, 1, 3, 4, 2, 4, 5};  // (a,c) -> packed symmetric index
  double* oS = P.outS + (size_t)prob * 9 * nq;
  double* oD = P.outD + (size_t)prob * 9 * nq;
  for (int j = threadIdx.x; j < nq; j += QT) {
    double r12[12];
#pragma unroll
    for (int q = 0; q < 12; ++q) r12[q] = 0.0;
    for (int b = 0; b < nb; ++b) {
      double av = P.A[(size_t)b * nq + j];
#pragma unroll
      for (int q = 0; q < 12; ++q) r12[q] = fma(Tm[q * nb + b], av, r12[q]);
    }
    if (P.kind == 1) {
      // subtract the coarse rule for source node j of sphere m (what the all-pairs kernel adds)
      double yx = tc[0] + P.a * P.xi[3 * j], yy = tc[1] + P.a * P.xi[3 * j + 1], yz = tc[2] + P.a * P.xi[3 * j + 2];
      double r0 = tx[0] - yx, r1 = tx[1] - yy, r2 = tx[2] - yz;
      double rr = r0 * r0 + r1 * r1 + r2 * r2;
      double ir = 1.0 / sqrt(rr), ir2 = ir * ir, ir3 = ir * ir2;
      double wq = P.w[j];
      double gs = cS * wq;
      r12[0] -= gs * (ir + r0 * r0 * ir3); r12[1] -= gs * r0 * r1 * ir3; r12[2] -= gs * r0 * r2 * ir3;
      r12[3] -= gs * (ir + r1 * r1 * ir3); r12[4] -= gs * r1 * r2 * ir3; r12[5] -= gs * (ir + r2 * r2 * ir3);
      double rn = r0 * P.xi[3 * j] + r1 * P.xi[3 * j + 1] + r2 * P.xi[3 * j + 2];
      double kd = cD * wq * rn * ir3 * ir2;
      r12[6] -= kd * r0 * r0; r12[7] -= kd * r0 * r1; r12[8] -= kd * r0 * r2;
      r12[9] -= kd * r1 * r1; r12[10] -= kd * r1 * r2; r12[11] -= kd * r2 * r2;
    }
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        if (P.want_s) oS[(size_t)a * 3 * nq + 3 * j + c] = r12[sym[3 * a + c]];
        oD[(size_t)a * 3 * nq + 3 * j + c] = r12[6 + sym[3 * a + c]];
      }
  }
}

// ------------------------------------------------------------------ near tensors by rotation
// The same refined near rule (R8) as k_quad_rows kind 1, evaluated in the frame F = [e1 e2 d]
// whose third axis d points from the source centre c_m to the target (the SH-
// rotation idea behind the "FFT-based acceleration of near-evaluation" of P:425):
//   * in that frame the target sits on the axis, x' = (0, 0, r'), and every kernel component
//     K'_ef(x', y'(theta', phi')) is a trigonometric polynomial of degree <= 2 in phi';
//   * the rule's 4p equispaced phi' nodes integrate (kernel) x (a degree-p SH) exactly, so only
//     the rotated basis functions with |m'| <= 2 see the kernel:  with the frame-rotated
//     coefficients D_b(m') of Y_b (Y_b(F eta') = sum_b' D_bb' Y_b'(eta'), b' of the same degree n),
//        T[b] = F M[b] F^T,   M_xx = D0 A_n + D2c B_n,  M_yy = D0 A_n - D2c B_n,  M_zz = D0 Z_n,
//                             M_xy = D2s B_n,  M_xz = D1c X_n,  M_yz = D1s X_n,
//     where A, Z, X, B are the theta'-rule integrals of the axisymmetric kernel factors times the
//     associated Legendre parts of degree n and order 0, 0, 1, 2 (4 (p+1) numbers per kernel);
//   * D_b(m') for |m'| <= 2 are read off second-order jets of the solid harmonic r^n Y_b at d
//     along e1, e2: value -> m' = 0, gradient -> m' = 1, traceless Hessian -> m' = 2 (every other
//     rotated mode vanishes to that order at the pole), divided by the same jets of the
//     reference functions at the pole (den[n][5], host).
// Cost O(p^2 + p n_theta) per incidence instead of the O(p^2 n_theta n_phi) of k_quad_rows (c4:
// 1.2 s -> milliseconds per geometry update); the values agree with k_quad_rows to rounding
// (GPU test) whenever n_phi > p + 2 (exactness of the phi' rule, checked by the caller).
struct Jet {  // second-order Taylor coefficients in (t1, t2): c0 + c1 t1 + c2 t2 + c11 t1^2 + c12 t1 t2 + c22 t2^2
  double c0, c1, c2, c11, c12, c22;
};
__host__ __device__ inline Jet jmul(const Jet& a, const Jet& b) {
  return Jet{a.c0 * b.c0,
             a.c0 * b.c1 + a.c1 * b.c0,
             a.c0 * b.c2 + a.c2 * b.c0,
             a.c0 * b.c11 + a.c1 * b.c1 + a.c11 * b.c0,
             a.c0 * b.c12 + a.c1 * b.c2 + a.c2 * b.c1 + a.c12 * b.c0,
             a.c0 * b.c22 + a.c2 * b.c2 + a.c22 * b.c0};
}
__host__ __device__ inline Jet jlin(const Jet& a, const Jet& l) {  // l linear (l.c11 = l.c12 = l.c22 = 0)
  return Jet{a.c0 * l.c0,
             a.c0 * l.c1 + a.c1 * l.c0,
             a.c0 * l.c2 + a.c2 * l.c0,
             a.c1 * l.c1 + a.c11 * l.c0,
             a.c1 * l.c2 + a.c2 * l.c1 + a.c12 * l.c0,
             a.c2 * l.c2 + a.c22 * l.c0};
}
__host__ __device__ inline Jet jaxpy(double s, const Jet& a, const Jet& b) {  // s a + b
  return Jet{fma(s, a.c0, b.c0), fma(s, a.c1, b.c1), fma(s, a.c2, b.c2),
             fma(s, a.c11, b.c11), fma(s, a.c12, b.c12), fma(s, a.c22, b.c22)};
}
__host__ __device__ inline Jet jscale(double s, const Jet& a) {
  return Jet{s * a.c0, s * a.c1, s * a.c2, s * a.c11, s * a.c12, s * a.c22};
}

// Jets of the solid harmonics of order m (cos and sin type, degrees l = m..lmax) at d along e1, e2
// (|d| = 1, e1, e2 orthonormal and orthogonal to d, so r^2 = 1 + t1^2 + t2^2); calls
// emit(l, jet_cos, jet_sin) for each l.  Same recurrences and normalisation as sh_column.
template <class Emit>
__host__ __device__ inline void solid_jets(int p, int lmax, int m, const double d[3], const double e1[3],
                                           const double e2[3], const double* ra, const double* rb,
                                           const double* cm, Emit emit) {
  const Jet X{d[0], e1[0], e2[0], 0, 0, 0}, Y{d[1], e1[1], e2[1], 0, 0, 0}, Z{d[2], e1[2], e2[2], 0, 0, 0};
  Jet re{1, 0, 0, 0, 0, 0}, im{0, 0, 0, 0, 0, 0};
  for (int k = 0; k < m; ++k) {  // (x + i y)^m
    const Jet a = jlin(re, X), b = jlin(im, Y), c = jlin(re, Y), e = jlin(im, X);
    re = jaxpy(-1.0, b, a);
    im = jaxpy(1.0, e, c);
  }
  const double s2 = 1.4142135623730951;
  const Jet cc = (m == 0) ? jscale(cm[0], re) : jscale(s2 * cm[m], re);
  const Jet ss = jscale(s2 * cm[m], im);
  Jet sm2{0, 0, 0, 0, 0, 0}, sm1{0, 0, 0, 0, 0, 0};
  for (int l = m; l <= lmax; ++l) {
    Jet s;
    if (l == m) {
      s = Jet{1, 0, 0, 0, 0, 0};
    } else if (l == m + 1) {
      s = jscale(ra[l * (p + 1) + m], jlin(sm1, Z));
    } else {  // r^(l-m) R_lm = a (z r^(l-1-m) R_{l-1,m} - b r^2 r^(l-2-m) R_{l-2,m})
      const Jet zs = jlin(sm1, Z);
      const Jet r2s{sm2.c0, sm2.c1, sm2.c2, sm2.c11 + sm2.c0, sm2.c12, sm2.c22 + sm2.c0};
      s = jscale(ra[l * (p + 1) + m], jaxpy(-rb[l * (p + 1) + m], r2s, zs));
    }
    sm2 = sm1;
    sm1 = s;
    emit(l, jmul(cc, s), jmul(ss, s));
  }
}

// den[n][5]: jets of the reference functions Y_n0, Y^c_n1, Y^s_n1, Y^c_n2, Y^s_n2 at the pole along x, y
// (value, d/dt1, d/dt2, the t1^2 - t2^2 and t1 t2 coefficients); zero where n < m'.
struct DenEmit {
  double* den;
  int m;
  __host__ __device__ void operator()(int l, const Jet& jc, const Jet& js) const {
    if (m == 0) den[5 * l] = jc.c0;
    if (m == 1) { den[5 * l + 1] = jc.c1; den[5 * l + 2] = js.c2; }
    if (m == 2) { den[5 * l + 3] = jc.c11 - jc.c22; den[5 * l + 4] = js.c12; }
  }
};
static void rot_denominators(int p, const std::vector<double>& ra, const std::vector<double>& rb,
                             const std::vector<double>& cm, std::vector<double>& den) {
  den.assign(5 * (size_t)(p + 1), 0.0);
  const double d[3] = {0, 0, 1}, e1[3] = {1, 0, 0}, e2[3] = {0, 1, 0};
  for (int m = 0; m <= std::min(2, p); ++m)
    solid_jets(p, p, m, d, e1, e2, ra.data(), rb.data(), cm.data(), DenEmit{den.data(), m});
}

struct RotParams {
  int p, nb, nbp, n1, n2;
  double a, mu, theta_c;
  const double *gl1_t, *gl1_w, *gl2_t, *gl2_w;
  const int *inc_t, *inc_m;
  const double *X, *centers;
  ShTables T;
  const double* den;  // [p+1][5]
  double *outS, *outD;  // [nprob][6][nbp]
  int want_s;
};

constexpr int NR_T = 128;
__global__ void __launch_bounds__(NR_T) k_near_rot(RotParams P) {
  extern __shared__ double rs[];
  const int p = P.p, nb = P.nb, nth = P.n1 + P.n2, pl = p + 1;
  double* Lg = rs;                  // [3][p+1][nth] Legendre parts of order 0, 1, 2
  double* fac = Lg + 3 * pl * nth;  // [8][nth] kernel factors x weights: S (A, Z, X, B), D (A, Z, X, B)
  double* W = fac + 8 * nth;        // [8][p+1]
  double* D5 = W + 8 * pl;          // [nb][5]
  int* degb = reinterpret_cast<int*>(D5 + 5 * (size_t)nb);  // [nb]
  __shared__ double F[9], rp, delta;
  const int prob = blockIdx.x, tid = threadIdx.x;
  if (tid == 0) {
    const int i = P.inc_t[prob], m = P.inc_m[prob];
    const double rx = P.X[3 * (size_t)i] - P.centers[3 * m], ry = P.X[3 * (size_t)i + 1] - P.centers[3 * m + 1],
                 rz = P.X[3 * (size_t)i + 2] - P.centers[3 * m + 2];
    const double r = sqrt(rx * rx + ry * ry + rz * rz);
    // frame from d = r / |r| with atan2 (acos loses ~1e-8 rad next to the poles)
    const double te = atan2(sqrt(rx * rx + ry * ry), rz), pe = atan2(ry, rx);
    const double ct = cos(te), st = sin(te), cp = cos(pe), sp = sin(pe);
    F[0] = cp * ct; F[1] = -sp; F[2] = cp * st;  // row-major: columns e1, e2, d
    F[3] = sp * ct; F[4] = cp;  F[5] = sp * st;
    F[6] = -st;     F[7] = 0.0; F[8] = ct;
    rp = r;
    delta = (r - P.a) / P.a;
  }
  __syncthreads();
  const double a = P.a, PI_ = PI;
  const double cS = 1.0 / (8.0 * PI_ * P.mu), cD = -3.0 / (4.0 * PI_);
  const double s2 = 1.4142135623730951;
  for (int k = tid; k < nth; k += NR_T) {
    double tt, ww;
    if (k < P.n1) {  // sinh-graded panel [0, theta_c] (R8)
      const double S = asinh(P.theta_c / delta);
      const double s = 0.5 * S * (P.gl1_t[k] + 1.0);
      tt = delta * sinh(s);
      ww = 0.5 * S * P.gl1_w[k] * delta * cosh(s);
    } else {
      const int kk = k - P.n1;
      tt = P.theta_c + 0.5 * (PI_ - P.theta_c) * (P.gl2_t[kk] + 1.0);
      ww = 0.5 * (PI_ - P.theta_c) * P.gl2_w[kk];
    }
    const double s = sin(tt), c = cos(tt), sh = sin(0.5 * tt);
    const double om = ww * s * a * a;
    const double rz = (rp - a) + 2.0 * a * sh * sh;  // r' - a cos(theta') without cancellation
    const double rho2 = a * a * s * s + rz * rz, ir = 1.0 / sqrt(rho2), ir2 = ir * ir, ir3 = ir * ir2;
    // Legendre parts R_l,m(cos theta'), m = 0, 1, 2, times cm, sqrt2 cm sin^m
    for (int m = 0; m <= 2; ++m) {
      const double pref = (m == 0) ? P.T.cm[0] : (m == 1 ? s2 * P.T.cm[1] * s : s2 * P.T.cm[2] * s * s);
      double rm2 = 0.0, rm1 = 0.0;
      for (int l = 0; l <= p; ++l) {
        double r = 0.0;
        if (l >= m && m <= p) {
          if (l == m) r = 1.0;
          else if (l == m + 1) r = P.T.ra[l * pl + m] * c;
          else r = P.T.ra[l * pl + m] * (c * rm1 - P.T.rb[l * pl + m] * rm2);
          rm2 = rm1;
          rm1 = r;
        }
        Lg[(m * pl + l) * nth + k] = pref * r;
      }
    }
    const double tp = 2.0 * PI_ * om, op = PI_ * om;  // phi' integrals: 2 pi (m' = 0), pi (m' >= 1)
    const double hs = 0.5 * a * a * s * s;
    fac[0 * nth + k] = tp * cS * (ir + hs * ir3);
    fac[1 * nth + k] = tp * cS * (ir + rz * rz * ir3);
    fac[2 * nth + k] = -op * cS * a * s * rz * ir3;
    fac[3 * nth + k] = op * cS * hs * ir3;
    const double kdf = cD * (rp * c - a) * ir3 * ir2;  // r.n_y = r' cos(theta') - a
    fac[4 * nth + k] = tp * kdf * hs;
    fac[5 * nth + k] = tp * kdf * rz * rz;
    fac[6 * nth + k] = -op * kdf * a * s * rz;
    fac[7 * nth + k] = op * kdf * hs;
  }
  __syncthreads();
  for (int e = tid; e < 8 * pl; e += NR_T) {  // W[q][l], theta' nodes summed in order
    const int q = e / pl, l = e - q * pl;
    const int mq = (q & 3) == 2 ? 1 : ((q & 3) == 3 ? 2 : 0);
    const double* L = Lg + (mq * pl + l) * nth;
    const double* f = fac + q * nth;
    double acc = 0.0;
    for (int k = 0; k < nth; ++k) acc = fma(f[k], L[k], acc);
    W[e] = acc;
  }
  if (tid <= p) {  // one order m per thread: rotated coefficients D5[b][m'] from the jets
    const int m = tid;
    const double d[3] = {F[2], F[5], F[8]}, e1[3] = {F[0], F[3], F[6]}, e2[3] = {F[1], F[4], F[7]};
    const double* den = P.den;
    solid_jets(p, p, m, d, e1, e2, P.T.ra, P.T.rb, P.T.cm, [&](int l, const Jet& jc, const Jet& js) {
      const double* dn = den + 5 * l;
      const double i0 = 1.0 / dn[0], i1 = l >= 1 ? 1.0 / dn[1] : 0.0, i2 = l >= 1 ? 1.0 / dn[2] : 0.0,
                   i3 = l >= 2 ? 1.0 / dn[3] : 0.0, i4 = l >= 2 ? 1.0 / dn[4] : 0.0;
      const int bc = sh_cos_index(p, l, m);
      double* o = D5 + 5 * bc;
      o[0] = jc.c0 * i0; o[1] = jc.c1 * i1; o[2] = jc.c2 * i2; o[3] = (jc.c11 - jc.c22) * i3; o[4] = jc.c12 * i4;
      degb[bc] = l;
      if (m >= 1 && m < p) {
        const int bs = sh_sin_index(p, l, m);
        o = D5 + 5 * bs;
        o[0] = js.c0 * i0; o[1] = js.c1 * i1; o[2] = js.c2 * i2; o[3] = (js.c11 - js.c22) * i3; o[4] = js.c12 * i4;
        degb[bs] = l;
      }
    });
  }
  __syncthreads();
  const int nbp = P.nbp;
  const size_t o = (size_t)prob * 6 * nbp;
  for (int b = tid; b < nbp; b += NR_T) {
    double tS[6] = {0, 0, 0, 0, 0, 0}, tD[6] = {0, 0, 0, 0, 0, 0};
    if (b < nb) {
      const int l = degb[b];
      const double* dv = D5 + 5 * b;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const double A = W[(4 * k) * pl + l], Zz = W[(4 * k + 1) * pl + l], Xx = W[(4 * k + 2) * pl + l],
                     B = W[(4 * k + 3) * pl + l];
        // M in the frame (symmetric), then T = F M F^T
        const double Mxx = fma(dv[0], A, dv[3] * B), Myy = fma(dv[0], A, -dv[3] * B), Mzz = dv[0] * Zz;
        const double Mxy = dv[4] * B, Mxz = dv[1] * Xx, Myz = dv[2] * Xx;
        double G[3][3];  // G = M F^T: G[e][c] = sum_f M[e][f] F[c][f]
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double f0 = F[3 * c], f1 = F[3 * c + 1], f2 = F[3 * c + 2];
          G[0][c] = Mxx * f0 + Mxy * f1 + Mxz * f2;
          G[1][c] = Mxy * f0 + Myy * f1 + Myz * f2;
          G[2][c] = Mxz * f0 + Myz * f1 + Mzz * f2;
        }
        double* t = k == 0 ? tS : tD;
        const int ia[6] = {0, 0, 0, 1, 1, 2}, ic[6] = {0, 1, 2, 1, 2, 2};  // xx, xy, xz, yy, yz, zz
#pragma unroll
        for (int q = 0; q < 6; ++q)
          t[q] = F[3 * ia[q]] * G[0][ic[q]] + F[3 * ia[q] + 1] * G[1][ic[q]] + F[3 * ia[q] + 2] * G[2][ic[q]];
      }
    }
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      P.outD[o + (size_t)q * nbp + b] = tD[q];
      if (P.want_s) P.outS[o + (size_t)q * nbp + b] = tS[q];
    }
  }
}

// ------------------------------------------------------------------ self expansion
// E_S[3i+a][3j+c] = (Rz(phi_l) Sring[k] Rz(phi_l)^T)[a][c] at j' = (k_j, l_j - l) - naive_S(i,j)
// E_L likewise with Dring and naive_D; E_A = E_L - I/2 + Pi_R.
__global__ void k_self_expand(int p, int nq, double a, double mu, const double* xi, const double* w,
                              const double* phi, const double* Sring, const double* Dring, double* ES,
                              double* EL, double* EA, double* EB, int want_s) {
  size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)nq * nq) return;
  int i = (int)(idx / nq), j = (int)(idx % nq);
  int tp = 2 * p;
  int ki = i / tp, li = i % tp;
  int kj = j / tp, lj = j % tp;
  int jr = kj * tp + ((lj - li) % tp + tp) % tp;
  double c = cos(phi[li]), s = sin(phi[li]);
  double Rz[9] = {c, -s, 0, s, c, 0, 0, 0, 1};
  const double PIl = 3.14159265358979323846;
  const double cS = 1.0 / (8.0 * PIl * mu), cD = -3.0 / (4.0 * PIl);
  double xi0 = a * xi[3 * i], xi1 = a * xi[3 * i + 1], xi2 = a * xi[3 * i + 2];
  double yj0 = a * xi[3 * j], yj1 = a * xi[3 * j + 1], yj2 = a * xi[3 * j + 2];
  double r[3] = {xi0 - yj0, xi1 - yj1, xi2 - yj2};
  double rr = r[0] * r[0] + r[1] * r[1] + r[2] * r[2];
  double nG[9] = {0}, nD[9] = {0};
  if (i != j) {
    double ir = 1.0 / sqrt(rr), ir3 = ir / rr;
    double rn = (r[0] * xi[3 * j] + r[1] * xi[3 * j + 1] + r[2] * xi[3 * j + 2]);
    for (int u = 0; u < 3; ++u)
      for (int v = 0; v < 3; ++v) {
        nG[3 * u + v] = cS * w[j] * ((u == v ? ir : 0.0) + r[u] * r[v] * ir3);
        nD[3 * u + v] = cD * w[j] * rn * r[u] * r[v] * ir3 / rr;
      }
  }
  for (int which = 0; which < 2; ++which) {
    if (which == 0 && !want_s) continue;
    const double* ring = (which == 0 ? Sring : Dring) + (size_t)ki * 9 * nq;
    double B[9];
    for (int u = 0; u < 3; ++u)
      for (int v = 0; v < 3; ++v) B[3 * u + v] = ring[(size_t)u * 3 * nq + 3 * jr + v];
    // Rz B Rz^T
    double T1[9], Rt[9];
    for (int u = 0; u < 3; ++u)
      for (int v = 0; v < 3; ++v) {
        double acc = 0;
        for (int q = 0; q < 3; ++q) acc += Rz[3 * u + q] * B[3 * q + v];
        T1[3 * u + v] = acc;
      }
    for (int u = 0; u < 3; ++u)
      for (int v = 0; v < 3; ++v) {
        double acc = 0;
        for (int q = 0; q < 3; ++q) acc += T1[3 * u + q] * Rz[3 * v + q];
        Rt[3 * u + v] = acc;
      }
    size_t ld = 3 * (size_t)nq;
    if (which == 0) {
      for (int u = 0; u < 3; ++u)
        for (int v = 0; v < 3; ++v) ES[(3 * (size_t)i + u) * ld + 3 * j + v] = Rt[3 * u + v] - nG[3 * u + v];
    } else {
      double ri_rj = xi0 * yj0 + xi1 * yj1 + xi2 * yj2;
      double ri[3] = {xi0, xi1, xi2}, rj[3] = {yj0, yj1, yj2};
      double cu = w[j] / (4.0 * PIl * a * a), co = 3.0 * w[j] / (8.0 * PIl * a * a * a * a);
      for (int u = 0; u < 3; ++u)
        for (int v = 0; v < 3; ++v) {
          double el = Rt[3 * u + v] - nD[3 * u + v];
          EL[(3 * (size_t)i + u) * ld + 3 * j + v] = el;
          double pir = (u == v ? cu + co * ri_rj : 0.0) - co * rj[u] * ri[v];
          double half = (i == j && u == v) ? 0.5 : 0.0;
          EA[(3 * (size_t)i + u) * ld + 3 * j + v] = el - half + pir;
          // the whole same-sphere block of A_op (D_self - I/2 + Pi_R), for the preconditioner
          if (EB) EB[(3 * (size_t)i + u) * ld + 3 * j + v] = Rt[3 * u + v] - half + pir;
        }
    }
  }
}

// ------------------------------------------------------------------ block-Jacobi inverse
// In-place Gauss-Jordan inversion with partial (row) pivoting of the n x n same-sphere
// block of A_op (identical for every sphere): per pivot column one single-CTA kernel
// (pivot search, row swap, row scaling, elimination factors) and one grid-wide rank-1
// elimination; column swaps undo the pivoting at the end.  Preconditioner of K4.
__global__ void k_gj_pivot(double* A, int n, int k, double* fcol, int* piv) {
  __shared__ double bv[1024];
  __shared__ int bi[1024];
  double best = -1.0;
  int bidx = k;
  for (int i = k + threadIdx.x; i < n; i += blockDim.x) {
    const double v = fabs(A[(size_t)i * n + k]);
    if (v > best) {
      best = v;
      bidx = i;
    }
  }
  bv[threadIdx.x] = best;
  bi[threadIdx.x] = bidx;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const double a = bv[threadIdx.x], b = bv[threadIdx.x + o];
      const int ia = bi[threadIdx.x], ib = bi[threadIdx.x + o];
      if (b > a || (b == a && ib < ia)) {
        bv[threadIdx.x] = b;
        bi[threadIdx.x] = ib;
      }
    }
    __syncthreads();
  }
  const int p = bi[0];
  if (threadIdx.x == 0) piv[k] = p;
  if (p != k)
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      const double t = A[(size_t)k * n + j];
      A[(size_t)k * n + j] = A[(size_t)p * n + j];
      A[(size_t)p * n + j] = t;
    }
  __syncthreads();
  const double d = 1.0 / A[(size_t)k * n + k];
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const double v = (j == k) ? 1.0 : A[(size_t)k * n + j];
    A[(size_t)k * n + j] = v * d;
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    fcol[i] = (i == k) ? 0.0 : A[(size_t)i * n + k];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (i != k) A[(size_t)i * n + k] = 0.0;
}

__global__ void k_gj_elim(double* A, int n, int k, const double* fcol) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (j >= n || i == k) return;
  const double f = fcol[i];
  if (f != 0.0) A[(size_t)i * n + j] = fma(-f, A[(size_t)k * n + j], A[(size_t)i * n + j]);
}

__global__ void k_gj_colswap(double* A, int n, const int* piv) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int k = n - 1; k >= 0; --k) {
    const int p = piv[k];
    if (p != k) {
      const double t = A[(size_t)i * n + k];
      A[(size_t)i * n + k] = A[(size_t)i * n + p];
      A[(size_t)i * n + p] = t;
    }
  }
}

void invert_in_place(double* A, int n, cudaStream_t st) {
  DBuf<double> fcol;
  DBuf<int> piv;
  fcol.alloc(n);
  piv.alloc(n);
  dim3 eg((n + 255) / 256, n);
  for (int k = 0; k < n; ++k) {
    k_gj_pivot<<<1, 1024, 0, st>>>(A, n, k, fcol.p, piv.p);
    k_gj_elim<<<eg, 256, 0, st>>>(A, n, k, fcol.p);
  }
  k_gj_colswap<<<(n + 127) / 128, 128, 0, st>>>(A, n, piv.p);
  BPQN_CHECK_LAUNCH();
  BPQN_CUDA(cudaStreamSynchronize(st));
}

// ------------------------------------------------------------------ driver
void precompute(Geom& g, cudaStream_t st, bool with_self) {
  const int p = g.p, nq = g.nq, nb = g.nb;
  BPQN_REQUIRE(3 * ((nb + 1) / 2) <= QT * 4, "p too large for k_quad_rows tiles (p <= 26)");
  BPQN_REQUIRE(g.nphi <= 256 && 2 * g.p_s <= 256 && g.n1 + g.n2 <= 128 && g.p_s + 1 <= 128,
               "quadrature node counts exceed kernel limits");
  std::vector<double> ra, rb, cm;
  sh_tables_host(p, ra, rb, cm);
  DBuf<double> d_ra, d_rb, d_cm;
  d_ra.alloc(ra.size()); d_rb.alloc(rb.size()); d_cm.alloc(cm.size());
  BPQN_CUDA(cudaMemcpyAsync(d_ra.p, ra.data(), ra.size() * 8, cudaMemcpyHostToDevice, st));
  BPQN_CUDA(cudaMemcpyAsync(d_rb.p, rb.data(), rb.size() * 8, cudaMemcpyHostToDevice, st));
  BPQN_CUDA(cudaMemcpyAsync(d_cm.p, cm.data(), cm.size() * 8, cudaMemcpyHostToDevice, st));
  ShTables T{d_ra.p, d_rb.p, d_cm.p};

  // analysis matrix
  if (with_self) {
  std::vector<double> wunit(nq);
  for (int i = 0; i < nq; ++i) wunit[i] = g.grid.w[i] / (g.a * g.a);
  DBuf<double> d_wunit, Yn;
  d_wunit.alloc(nq);
  Yn.alloc((size_t)nb * nq);
  BPQN_CUDA(cudaMemcpyAsync(d_wunit.p, wunit.data(), nq * 8, cudaMemcpyHostToDevice, st));
  g.analysis.alloc((size_t)nb * nq);
  k_analysis<<<(nq + 127) / 128, 128, 0, st>>>(p, nq, g.xi_d.p, d_wunit.p, T, Yn.p, g.analysis.p, nb);
  BPQN_CHECK_LAUNCH();
  BPQN_CUDA(cudaStreamSynchronize(st));  // d_wunit / Yn are released at the end of this scope
  }

  // GL tables
  std::vector<double> t_s, w_s, t1, w1, t2, w2;
  gauss_legendre_desc(g.p_s + 1, t_s, w_s);
  gauss_legendre_desc(g.n1, t1, w1);
  gauss_legendre_desc(g.n2, t2, w2);
  DBuf<double> dts, dws, dt1, dw1, dt2, dw2, dth;
  auto up = [&](DBuf<double>& d, const std::vector<double>& h) {
    d.alloc(h.size());
    BPQN_CUDA(cudaMemcpyAsync(d.p, h.data(), h.size() * 8, cudaMemcpyHostToDevice, st));
  };
  up(dts, t_s); up(dws, w_s); up(dt1, t1); up(dw1, w1); up(dt2, t2); up(dw2, w2); up(dth, g.grid.theta);
  DBuf<double> dphi;
  up(dphi, g.grid.phi);

  QuadParams P{};
  P.p = p; P.nq = nq; P.nb = nb; P.a = g.a; P.mu = g.mu;
  P.ns_t = g.p_s + 1; P.ns_p = 2 * g.p_s;
  P.gl_self_t = dts.p; P.gl_self_w = dws.p; P.theta_ring = dth.p;
  P.n1 = g.n1; P.n2 = g.n2; P.nphi = g.nphi; P.theta_c = 1.0;
  P.gl1_t = dt1.p; P.gl1_w = dw1.p; P.gl2_t = dt2.p; P.gl2_w = dw2.p;
  P.X = g.X.p; P.centers = g.centers_d.p;
  P.xi = g.xi_d.p; P.w = g.w_d.p; P.A = g.analysis.p; P.T = T;
  size_t smem = (128 + 128 + 128 + 256 + 256 + QPC * 12 + (size_t)QPC * nb + 12 * (size_t)nb) * sizeof(double);
  BPQN_CUDA(cudaFuncSetAttribute(k_quad_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));

  // self rings (depend on p, a, mu only: kept by bpqn_geometry_update)
  if (with_self) {
  DBuf<double> Sring, Dring;
  Sring.alloc((size_t)(p + 1) * 9 * nq);
  Dring.alloc((size_t)(p + 1) * 9 * nq);
  P.kind = 0; P.outS = Sring.p; P.outD = Dring.p; P.want_s = 1;
  k_quad_rows<<<p + 1, QT, smem, st>>>(P);
  BPQN_CHECK_LAUNCH();
  size_t ne = (size_t)3 * nq * 3 * nq;
  if (g.single_layer) g.E_S.alloc(ne);
  g.E_L.alloc(ne);
  g.E_A.alloc(ne);
  g.Minv.alloc(ne);
  size_t nn = (size_t)nq * nq;
  k_self_expand<<<(unsigned)((nn + 255) / 256), 256, 0, st>>>(p, nq, g.a, g.mu, g.xi_d.p, g.w_d.p, dphi.p,
                                                             Sring.p, Dring.p, g.E_S.p, g.E_L.p, g.E_A.p, g.Minv.p,
                                                             g.single_layer ? 1 : 0);
  BPQN_CHECK_LAUNCH();
  invert_in_place(g.Minv.p, 3 * nq, st);
  }

  // near incidences, in K2 order (by source sphere)
  g.T_D.release();
  g.T_S.release();
  if (g.n_inc > 0) {
    size_t per = (size_t)6 * ((nb + 1) & ~1);
    g.T_D.alloc((size_t)g.n_inc * per);
    if (g.single_layer) g.T_S.alloc((size_t)g.n_inc * per);
    P.kind = 1; P.inc_t = g.cm_t.p; P.inc_m = g.cm_m.p;
    P.want_s = g.single_layer ? 1 : 0;
    // the rotation form needs an exact phi' rule for (kernel, degree <= 2) x (degree <= p)
    const char* eb = getenv("BPQN_NEAR_BRUTE");
    const bool rot = g.nphi > p + 2 && !(eb && eb[0] == '1');
    if (rot) {
      std::vector<double> den;
      rot_denominators(p, ra, rb, cm, den);
      DBuf<double> dden;
      up(dden, den);
      RotParams R{};
      R.p = p; R.nb = nb; R.nbp = (nb + 1) & ~1; R.n1 = g.n1; R.n2 = g.n2;
      R.a = g.a; R.mu = g.mu; R.theta_c = 1.0;
      R.gl1_t = dt1.p; R.gl1_w = dw1.p; R.gl2_t = dt2.p; R.gl2_w = dw2.p;
      R.X = g.X.p; R.centers = g.centers_d.p; R.T = T; R.den = dden.p;
      R.want_s = P.want_s;
      const int nth = g.n1 + g.n2;
      const size_t rsm = (3 * (size_t)(p + 1) * nth + 8 * (size_t)nth + 8 * (size_t)(p + 1) + 5 * (size_t)nb) * 8 +
                         4 * (size_t)nb;
      BPQN_CUDA(cudaFuncSetAttribute(k_near_rot, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm));
      const long long batch = 1 << 20;
      for (long long b0 = 0; b0 < g.n_inc; b0 += batch) {
        const long long nbt = std::min(batch, g.n_inc - b0);
        RotParams Q = R;
        Q.inc_t = g.cm_t.p + b0;
        Q.inc_m = g.cm_m.p + b0;
        Q.outD = g.T_D.p + b0 * per;
        Q.outS = g.single_layer ? g.T_S.p + b0 * per : nullptr;
        k_near_rot<<<(unsigned)nbt, NR_T, rsm, st>>>(Q);
        BPQN_CHECK_LAUNCH();
      }
      BPQN_CUDA(cudaStreamSynchronize(st));  // dden is released at the end of this scope
      return;
    }
    // batch to keep grids modest
    const long long batch = 65535;
    for (long long b0 = 0; b0 < g.n_inc; b0 += batch) {
      long long nbt = std::min(batch, g.n_inc - b0);
      QuadParams Q = P;
      Q.inc_t = g.cm_t.p + b0;
      Q.inc_m = g.cm_m.p + b0;
      Q.outD = g.T_D.p + b0 * per;
      Q.outS = g.single_layer ? g.T_S.p + b0 * per : g.T_D.p + b0 * per;  // unused when !want_s
      k_quad_rows<<<(unsigned)nbt, QT, smem, st>>>(Q);
      BPQN_CHECK_LAUNCH();
    }
  }
  BPQN_CUDA(cudaStreamSynchronize(st));
}

}  // namespace bpqn
