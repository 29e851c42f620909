/* Oracle direct Stokes sums -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
 *
 * Plain double loop, fp64, OpenMP over targets.  Computes, for every target i,
 *
 *   u_i = sum_j w_j [ G(x_i - y_j) f_j + K_D(x_i, y_j) q_j ]
 *
 *   G(r)      = 1/(8 pi mu) (I/rho + r r^T/rho^3)
 *   K_D(x, y) = -3/(4 pi) (r . n_y) r r^T / rho^5,      r = x - y
 *
 * (reading R3 / O3, O6 of SURVEY 8(c); the paper treats the Stokes solver as a
 * black box).  f or q may be NULL.  The caller
 * passes only source sets that exclude the target's own sphere; a pair with
 * rho == 0 is counted in the return value and skipped.
 */
#include <math.h>
#include <stddef.h>

long oracle_direct_sum(long nt, const double* x, long ns, const double* y,
                       const double* ny, const double* w, const double* f,
                       const double* q, double mu, double* u) {
  const double cS = 1.0 / (8.0 * M_PI * mu);
  const double cD = -3.0 / (4.0 * M_PI);
  long nzero = 0;
#pragma omp parallel for schedule(static) reduction(+ : nzero)
  for (long i = 0; i < nt; ++i) {
    double u0 = 0.0, u1 = 0.0, u2 = 0.0;
    const double x0 = x[3 * i], x1 = x[3 * i + 1], x2 = x[3 * i + 2];
    for (long j = 0; j < ns; ++j) {
      const double r0 = x0 - y[3 * j], r1 = x1 - y[3 * j + 1], r2 = x2 - y[3 * j + 2];
      const double rho2 = r0 * r0 + r1 * r1 + r2 * r2;
      if (rho2 == 0.0) { nzero += 1; continue; }
      const double rho = sqrt(rho2);
      const double irho = 1.0 / rho;
      const double irho3 = irho / rho2;
      const double wj = w[j];
      if (f) {
        const double f0 = f[3 * j], f1 = f[3 * j + 1], f2 = f[3 * j + 2];
        const double rf = r0 * f0 + r1 * f1 + r2 * f2;
        u0 += cS * wj * (f0 * irho + r0 * rf * irho3);
        u1 += cS * wj * (f1 * irho + r1 * rf * irho3);
        u2 += cS * wj * (f2 * irho + r2 * rf * irho3);
      }
      if (q) {
        const double n0 = ny[3 * j], n1 = ny[3 * j + 1], n2 = ny[3 * j + 2];
        const double q0 = q[3 * j], q1 = q[3 * j + 1], q2 = q[3 * j + 2];
        const double rn = r0 * n0 + r1 * n1 + r2 * n2;
        const double rq = r0 * q0 + r1 * q1 + r2 * q2;
        const double irho5 = irho3 / rho2;
        const double t = cD * wj * rn * rq * irho5;
        u0 += t * r0;
        u1 += t * r1;
        u2 += t * r2;
      }
    }
    u[3 * i] = u0;
    u[3 * i + 1] = u1;
    u[3 * i + 2] = u2;
  }
  return nzero;
}

/* Far (coarse-rule) part of the layer operator O6 with per-target exclusions:
 * target t lies on sphere tsph[t]; spheres excl[excl_ptr[t] .. excl_ptr[t+1])
 * are near to it (handled by the refined rule) and skipped, as is its own sphere.
 * Sources are the nq nodes of every other sphere m (node index m*nq + j). */
long oracle_far_sum(long nt, const double* x, const long* tsph, const long* excl_ptr,
                    const long* excl, long nsph, long nq, const double* y,
                    const double* ny, const double* w, const double* f,
                    const double* q, double mu, double* u) {
  const double cS = 1.0 / (8.0 * M_PI * mu);
  const double cD = -3.0 / (4.0 * M_PI);
  long nzero = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(+ : nzero)
  for (long t = 0; t < nt; ++t) {
    double u0 = 0.0, u1 = 0.0, u2 = 0.0;
    const double x0 = x[3 * t], x1 = x[3 * t + 1], x2 = x[3 * t + 2];
    for (long m = 0; m < nsph; ++m) {
      if (m == tsph[t]) continue;
      int skip = 0;
      for (long e = excl_ptr[t]; e < excl_ptr[t + 1]; ++e)
        if (excl[e] == m) skip = 1;
      if (skip) continue;
      for (long j = m * nq; j < (m + 1) * nq; ++j) {
        const double r0 = x0 - y[3 * j], r1 = x1 - y[3 * j + 1], r2 = x2 - y[3 * j + 2];
        const double rho2 = r0 * r0 + r1 * r1 + r2 * r2;
        if (rho2 == 0.0) { nzero += 1; continue; }
        const double rho = sqrt(rho2);
        const double irho = 1.0 / rho;
        const double irho3 = irho / rho2;
        const double wj = w[j];
        if (f) {
          const double f0 = f[3 * j], f1 = f[3 * j + 1], f2 = f[3 * j + 2];
          const double rf = r0 * f0 + r1 * f1 + r2 * f2;
          u0 += cS * wj * (f0 * irho + r0 * rf * irho3);
          u1 += cS * wj * (f1 * irho + r1 * rf * irho3);
          u2 += cS * wj * (f2 * irho + r2 * rf * irho3);
        }
        if (q) {
          const double n0 = ny[3 * j], n1 = ny[3 * j + 1], n2 = ny[3 * j + 2];
          const double q0 = q[3 * j], q1 = q[3 * j + 1], q2 = q[3 * j + 2];
          const double rn = r0 * n0 + r1 * n1 + r2 * n2;
          const double rq = r0 * q0 + r1 * q1 + r2 * q2;
          const double t5 = cD * wj * rn * rq * irho3 / rho2;
          u0 += t5 * r0;
          u1 += t5 * r1;
          u2 += t5 * r2;
        }
      }
    }
    u[3 * t] = u0;
    u[3 * t + 1] = u1;
    u[3 * t + 2] = u2;
  }
  return nzero;
}
