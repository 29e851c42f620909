"""Pins for the oracle's grid, SH projection, self and near quadrature (not gpu).

Each test checks the oracle against something other than itself: closed-form
sphere moments (P1), a library SH routine (scipy), the Stokes closed forms on and
off a sphere (App. A.1 of SURVEY; P3, P4, P6), and convergence against finer rules.
"""
import math

import numpy as np
import pytest
import scipy.special as sps

from oracle.grid import sphere_grid
from oracle.nearquad import near_points, near_rule
from oracle.sh import Projector, basis_lm, norm_legendre, real_sh
from oracle.stokes import self_rows, stokeslet, stresslet


def sphere_moment(a, b, c):
    """int_{S^2} x^a y^b z^c dS (closed form)."""
    if a % 2 or b % 2 or c % 2:
        return 0.0
    g = math.gamma
    return 2.0 * g((a + 1) / 2) * g((b + 1) / 2) * g((c + 1) / 2) / g((a + b + c + 3) / 2)


@pytest.mark.parametrize("p", [4, 8, 12])
def test_grid_moments(p):
    g = sphere_grid(p, a=1.7)
    assert abs(g["w"].sum() - 4 * np.pi * 1.7 ** 2) < 1e-13 * 4 * np.pi * 1.7 ** 2
    g1 = sphere_grid(p)
    x, y, z = g1["xi"].T
    for deg in range(0, 2 * p):  # trapezoid(2p) exact for |m| < 2p, GL(p+1) to 2p+1
        for a in range(deg + 1):
            for b in range(deg + 1 - a):
                c = deg - a - b
                got = np.sum(g1["w"] * x ** a * y ** b * z ** c)
                assert abs(got - sphere_moment(a, b, c)) < 1e-13, (a, b, c)


def test_legendre_vs_scipy():
    rng = np.random.default_rng(0)
    xyz = rng.standard_normal((50, 3))
    xyz /= np.linalg.norm(xyz, axis=1, keepdims=True)
    p = 12
    Y = real_sh(p, xyz)
    th = np.arccos(xyz[:, 2])
    ph = np.arctan2(xyz[:, 1], xyz[:, 0])
    for k, (l, m) in enumerate(basis_lm(p)):
        Yc = sps.sph_harm_y(l, abs(m), th, ph)
        if m == 0:
            ref = Yc.real
        elif m > 0:
            ref = np.sqrt(2.0) * Yc.real
        else:
            ref = np.sqrt(2.0) * Yc.imag
        # sign conventions (Condon-Shortley) may differ: compare up to a global sign
        s = np.sign(np.dot(ref, Y[:, k]))
        assert np.abs(s * Y[:, k] - ref).max() < 1e-12, (l, m)


def test_sh_orthonormal_and_nyquist():
    p = 10
    hi = sphere_grid(3 * p)
    Y = real_sh(p, hi["xi"])
    gram = Y.T @ (Y * hi["w"][:, None])
    assert np.abs(gram - np.eye(gram.shape[0])).max() < 1e-12
    g = sphere_grid(p)
    Yg = real_sh(p, g["xi"])
    gram_d = Yg.T @ (Yg * g["w"][:, None])
    expect = np.eye(gram.shape[0])
    k = basis_lm(p).index((p, p))
    expect[k, k] = 2.0          # App. A.3: discrete norm of cos(p phi) is twice the continuous one
    assert np.abs(gram_d - expect).max() < 1e-12


@pytest.mark.parametrize("p", [6, 9])
def test_projection(p):
    g = sphere_grid(p)
    pr = Projector(g)
    P = pr.matrix()
    rng = np.random.default_rng(1)
    c = rng.standard_normal(len(basis_lm(p)))
    v = real_sh(p, g["xi"]) @ c
    assert np.abs(P @ v - v).max() < 1e-12           # reproduces V_p
    z = rng.standard_normal(g["xi"].shape[0])
    assert np.abs(P @ (P @ z) - P @ z).max() < 1e-12  # idempotent
    th, ph = g["theta_node"], g["phi_node"]
    s = np.sin(p * ph) * np.sin(th) ** p              # sin(p phi) P_p^p, zero on the grid
    assert np.abs(s).max() < 1e-12
    # interpolation at off-grid points reproduces V_p too
    pts = rng.standard_normal((20, 3))
    pts /= np.linalg.norm(pts, axis=1, keepdims=True)
    assert np.abs(pr.interp_rows(pts) @ v - real_sh(p, pts) @ c).max() < 1e-12


@pytest.mark.parametrize("p", [8, 16])
def test_self_closed_forms(p):
    """P3/P4: S[const] = 2a/(3mu) const, S[rot traction] = Omega x x, S[xi] = 0,
    D[const] = const/2, D[rigid] = rigid/2, D[xi] = -xi/2 (on the surface)."""
    a, mu = 1.3, 0.7
    g = sphere_grid(p, a)
    pr = Projector(g)
    nq = g["xi"].shape[0]
    f0 = np.array([0.3, -0.7, 1.1])
    T = np.array([0.2, 0.5, -0.4])
    Om = np.array([0.3, 0.1, -0.2])
    for i in [0, nq // 3, nq - 1]:
        S, D = self_rows(g, pr, i, 2 * p, mu)
        x = a * g["xi"][i]
        ap = lambda M, v: np.einsum("ajb,jb->a", M, v)
        assert np.abs(ap(S, np.tile(f0, (nq, 1))) - 2 * a / (3 * mu) * f0).max() < 1e-12
        fr = 3 / (8 * np.pi * a ** 3) * np.cross(T, g["xi"])
        assert np.abs(ap(S, fr) - np.cross(T / (8 * np.pi * mu * a ** 3), x)).max() < 1e-12
        assert np.abs(ap(S, g["xi"])).max() < 1e-12
        assert np.abs(ap(D, np.tile(f0, (nq, 1))) - 0.5 * f0).max() < 1e-12
        rr = np.cross(Om, a * g["xi"])
        assert np.abs(ap(D, rr) - 0.5 * rr[i]).max() < 1e-12
        assert np.abs(ap(D, g["xi"]) + 0.5 * g["xi"][i]).max() < 1e-12


def test_self_converged_in_ps():
    """R6: p_s = 2p agrees with p_s = 4p to <= 1e-10 on a random V_p density."""
    p = 12
    g = sphere_grid(p)
    pr = Projector(g)
    rng = np.random.default_rng(2)
    sig = pr.matrix() @ rng.standard_normal((g["xi"].shape[0], 3))
    for i in [5, 77]:
        A = self_rows(g, pr, i, 2 * p, 1.0)
        B = self_rows(g, pr, i, 4 * p, 1.0)
        for k in range(2):
            u1 = np.einsum("ajb,jb->a", A[k], sig)
            u2 = np.einsum("ajb,jb->a", B[k], sig)
            assert np.abs(u1 - u2).max() < 1e-10


def exact_translating_rotating(x, F, T, mu):
    r = x
    rho = np.linalg.norm(r)
    I = np.eye(3)
    G = (I / rho + np.outer(r, r) / rho ** 3 + (1 / 3) * (I / rho ** 3 - 3 * np.outer(r, r) / rho ** 5)) / (8 * np.pi * mu)
    return G @ F + np.cross(T, r) / rho ** 3 / (8 * np.pi * mu)


@pytest.mark.parametrize("p", [8, 16])
@pytest.mark.parametrize("h", [1e-4, 1e-2, 0.3])
def test_near_rule_exterior_closed_forms(p, h):
    """P6 near the surface: S[P^T(F,T)] = exact moving-sphere field, D[const] = 0."""
    mu = 1.0
    F = np.array([0.3, -0.5, 0.8])
    T = np.array([0.1, 0.7, -0.2])
    rule = near_rule(p)
    for dn in [np.array([0.3, 0.2, 0.9]), np.array([0.0, 0.0, -1.0]), np.array([0.6, -0.64, 0.1])]:
        x = (1 + h) * dn / np.linalg.norm(dn)
        eta, w = near_points(x, np.zeros(3), 1.0, rule)
        r = x[None] - eta
        f = F / (4 * np.pi) + 3 / (8 * np.pi) * np.cross(T, eta)
        u = np.einsum("sab,sb->a", stokeslet(r, mu) * w[:, None, None], f)
        ex = exact_translating_rotating(x, F, T, mu)
        assert np.abs(u - ex).max() < 1e-12 * max(1.0, np.abs(ex).max())
        ud = np.einsum("sab,b->a", stresslet(r, eta) * w[:, None, None], np.array([1.0, 2, 3]))
        assert np.abs(ud).max() < 1e-11


def test_near_rule_converged_random_density():
    """The refined rule on a random V_p density agrees with a 2x finer rule."""
    p = 12
    g = sphere_grid(p)
    pr = Projector(g)
    rng = np.random.default_rng(3)
    sig = pr.matrix() @ rng.standard_normal((g["xi"].shape[0], 3))
    fine = dict(n1=4 * p + 32, n2=2 * p + 16, nphi=8 * p, theta_c=1.0)
    for h in [1e-3, 0.05, 0.8]:
        x = (1 + h) * np.array([0.48, -0.6, 0.64])
        vals = []
        for rule in (near_rule(p), fine):
            eta, w = near_points(x, np.zeros(3), 1.0, rule)
            r = x[None] - eta
            s = pr.interp_rows(eta) @ sig
            vals.append(np.einsum("sab,sb->a", (stokeslet(r, 1.0) + stresslet(r, eta)) * w[:, None, None], s))
        assert np.abs(vals[0] - vals[1]).max() < 1e-11 * np.abs(vals[1]).max()


def test_legendre_recurrence_small_closed_forms():
    t = np.linspace(-1, 1, 7)
    P = norm_legendre(2, t)
    assert np.allclose(P[0, 0], 1 / np.sqrt(2))
    assert np.allclose(P[1, 0], np.sqrt(1.5) * t)
    assert np.allclose(np.abs(P[1, 1]), np.sqrt(0.75) * np.sqrt(1 - t * t))
