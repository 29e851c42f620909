"""Near-singular quadrature for targets close to another sphere (oracle; TEST INFRASTRUCTURE ONLY).

Reading R8 (replaces SURVEY R8's plain 2x upsampling, which gave
wrong-sign two-sphere mobilities at gap 0.1, p = 12): the paper names the near
evaluation only as O(p^4) / FFT-accelerated.  Definition:

* near incidence: target x (on sphere n) and source sphere m != n with
  h = |x - c_m| - a < d_near = 4 pi a / p;
* refined rule on sphere m: a polar grid whose pole is the point of sphere m
  closest to x, e = (x - c_m)/|x - c_m| = (sin te cos pe, sin te sin pe, cos te),
  rotation R = R_z(pe) R_y(te);
    theta' panel 1: theta' = delta sinh(s), delta = h/a, s in [0, asinh(theta_c/delta)],
                    n1 = 2p + 16 Gauss-Legendre nodes in s, theta_c = 1 rad;
    theta' panel 2: theta' in [theta_c, pi], n2 = p + 8 Gauss-Legendre nodes;
    phi' = 2 pi l / (4p), l = 0..4p-1;
    weight a^2 sin(theta') w_theta' (2 pi / 4p);
  the density there is the Pi_p interpolant of sphere m's nodal density.
* the refined rule REPLACES the coarse nodal sum over sphere m for that target.

Accuracy (tests/test_oracle_geometry.py: test_near_rule_exterior_closed_forms,
test_near_rule_converged_random_density): the exterior closed forms (translating /
rotating sphere field for S, D[const] = 0 outside) hold to <= 1e-12 for
h in [1e-4, d_near], and a random V_p density agrees with a 4x finer rule.
"""
import numpy as np

from .grid import gauss_legendre
from .sh import real_sh
from .stokes import rot_y, rot_z, stokeslet, stresslet

THETA_C = 1.0


def near_rule(p):
    return dict(n1=2 * p + 16, n2=p + 8, nphi=4 * p, theta_c=THETA_C)


def near_points(x, c, a, rule):
    """Unit points (relative to sphere m, [n_s,3]) and area weights [n_s] of the
    refined rule for target x near the sphere (c, a)."""
    rel = np.asarray(x, dtype=np.float64) - np.asarray(c, dtype=np.float64)
    d = np.linalg.norm(rel)
    e = rel / d
    delta = (d - a) / a
    te = np.arccos(np.clip(e[2], -1.0, 1.0))
    pe = np.arctan2(e[1], e[0])
    R = rot_z(pe) @ rot_y(te)
    thc = rule["theta_c"]
    t1, o1 = gauss_legendre(rule["n1"])
    S = np.arcsinh(thc / delta)
    s = 0.5 * S * (t1 + 1.0)
    th1 = delta * np.sinh(s)
    w1 = 0.5 * S * o1 * delta * np.cosh(s)
    t2, o2 = gauss_legendre(rule["n2"])
    th2 = thc + 0.5 * (np.pi - thc) * (t2 + 1.0)
    w2 = 0.5 * (np.pi - thc) * o2
    th = np.concatenate([th1, th2])
    wth = np.concatenate([w1, w2]) * np.sin(th)
    nphi = rule["nphi"]
    ph = 2.0 * np.pi * np.arange(nphi) / nphi
    TH, PH = np.meshgrid(th, ph, indexing="ij")
    eta = np.stack([np.sin(TH) * np.cos(PH), np.sin(TH) * np.sin(PH), np.cos(TH)], axis=-1).reshape(-1, 3)
    wts = a * a * np.outer(wth, np.full(nphi, 2.0 * np.pi / nphi)).reshape(-1)
    return eta @ R.T, wts


def near_tensor(x, c, a, mu, p, rule=None):
    """T[kind, alpha, beta, b] = sum_s w_s K_kind(x - y_s)[alpha, beta] Y_b(eta_s),
    kind 0 = Stokeslet G, 1 = stresslet K_D (n_y = eta_s).  The refined-rule
    contribution of sphere m at x is then sum_b T[kind, :, :, b] @ coef_b where
    coef = SH coefficients of the density's Pi_p interpolant (Projector.analysis)."""
    rule = near_rule(p) if rule is None else rule
    eta, wts = near_points(x, c, a, rule)
    y = np.asarray(c) + a * eta
    r = np.asarray(x)[None, :] - y
    Y = real_sh(p, eta)                                  # [n_s, nb]
    G = stokeslet(r, mu) * wts[:, None, None]
    K = stresslet(r, eta) * wts[:, None, None]
    return np.stack([np.einsum("sab,sk->abk", G, Y), np.einsum("sab,sk->abk", K, Y)])


def incidences(X, sphere_of, centers, a, dnear, pairs):
    """List of (target global index i, source sphere m) with h < dnear, restricted
    to sphere pairs in ``pairs`` (the candidate (n, m) with gap < dnear)."""
    out = []
    nq = X.shape[0] // centers.shape[0]
    for (n, m) in pairs:
        for (tn, sm) in ((n, m), (m, n)):
            xs = X[tn * nq:(tn + 1) * nq]
            h = np.linalg.norm(xs - centers[sm], axis=1) - a
            for k in np.nonzero(h < dnear)[0]:
                out.append((tn * nq + int(k), sm))
    out.sort()
    return out
