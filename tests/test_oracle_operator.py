"""Pins for the oracle's layer operator, mobility and LCP operator (not gpu).

P5: the C far sum against an extended-precision numpy brute force.
P6: far-field closed forms through the whole layer operator.
P7: single-sphere drag, single Janus sphere, GMRES vs a dense solve, exact
    covariance under the grid's z-rotation by pi/p, far spheres vs RPY.
P8: D column = finite difference of the gap; D^T of a common translation = 0;
    A = D^T M D symmetric to discretisation error and positive definite.
"""
import numpy as np
import pytest

from oracle import lcp, mobility as mob, native
from oracle.layer import Disc
from oracle.stokes import rot_z


def longdouble_sum(x, y, ny, w, f, q, mu):
    L = np.longdouble
    x, y, ny, w, f, q = (np.asarray(v, dtype=L) for v in (x, y, ny, w, f, q))
    out = np.zeros((x.shape[0], 3), dtype=L)
    pi = L(np.pi)
    for i in range(x.shape[0]):
        r = x[i] - y
        rho2 = (r * r).sum(axis=1)
        rho = np.sqrt(rho2)
        rf = (r * f).sum(axis=1)
        rn = (r * ny).sum(axis=1)
        rq = (r * q).sum(axis=1)
        s = w[:, None] * (f / rho[:, None] + r * (rf / rho ** 3)[:, None]) / (8 * pi * L(mu))
        d = -L(3) / (4 * pi) * w[:, None] * r * (rn * rq / rho ** 5)[:, None]
        out[i] = (s + d).sum(axis=0)
    return out


def test_direct_sum_vs_longdouble():
    rng = np.random.default_rng(5)
    x = rng.standard_normal((17, 3)) * 3
    y = rng.standard_normal((300, 3))
    ny = rng.standard_normal((300, 3))
    w = rng.uniform(0.1, 1, 300)
    f = rng.standard_normal((300, 3))
    q = rng.standard_normal((300, 3))
    u = native.direct_sum(x, y, ny, w, f, q, 0.8)
    ref = longdouble_sum(x, y, ny, w, f, q, 0.8).astype(np.float64)
    assert np.abs(u - ref).max() < 1e-13 * np.abs(ref).max()
    # far_sum with sphere exclusions == direct_sum on the kept sources
    nq = 30
    tsph = np.full(17, 3)
    ptr = np.arange(0, 18) // 2 * 0
    ptr = np.zeros(18, dtype=np.int64)
    u2 = native.far_sum(x, tsph, ptr, np.zeros(0, dtype=np.int64), 10, nq, y, ny, w, f, q, 0.8)
    keep = np.ones(300, dtype=bool)
    keep[3 * nq:4 * nq] = False
    u3 = native.direct_sum(x, y[keep], ny[keep], w[keep], f[keep], q[keep], 0.8)
    assert np.abs(u2 - u3).max() < 1e-14 * np.abs(u3).max()


def two_spheres(gap, p, d=np.array([1.0, 0.3, -0.2])):
    d = d / np.linalg.norm(d)
    return Disc(np.array([[0.1, -0.2, 0.3], [0.1, -0.2, 0.3] + (2 + gap) * d]), p)


def test_layer_far_field_and_gauss():
    """P6 through L: S[P^T(F,T)] on sphere 1 seen at sphere 0's nodes equals the
    exact translating/rotating-sphere field; D[const on sphere 1] = 0 there;
    D[const on sphere 0] = const/2 on sphere 0 (Gauss, PV)."""
    for gap, p in [(0.05, 8), (1.0, 8), (0.3, 12)]:
        dsc = two_spheres(gap, p)
        FT = np.zeros((2, 6))
        FT[1] = [0.3, -0.5, 0.8, 0.1, 0.7, -0.2]
        f = mob.PT(dsc, FT)
        u = dsc.apply_all(f=f)[: dsc.nq]
        c1 = dsc.centers[1]
        for i in range(0, dsc.nq, 7):
            r = dsc.X[i] - c1
            rho = np.linalg.norm(r)
            I = np.eye(3)
            G = (I / rho + np.outer(r, r) / rho ** 3 + (I / rho ** 3 - 3 * np.outer(r, r) / rho ** 5) / 3) / (8 * np.pi)
            ex = G @ FT[1, :3] + np.cross(FT[1, 3:], r) / rho ** 3 / (8 * np.pi)
            h = rho - 1
            tol = 1e-11 if h < dsc.dnear else 1e-4     # coarse rule beyond d_near: discretisation error
            assert np.abs(u[i] - ex).max() < tol * max(1, np.abs(ex).max()), (gap, p, i, h)
        q = np.zeros((dsc.N, 3))
        q[dsc.nq:] = [1.0, -2.0, 0.5]
        v = dsc.apply_all(q=q)
        near0 = np.array([len(e) > 0 for e in dsc.excl[: dsc.nq]])
        assert np.abs(v[: dsc.nq][near0]).max() < 1e-11
        q2 = np.zeros((dsc.N, 3))
        q2[: dsc.nq] = [1.0, -2.0, 0.5]
        v2 = dsc.apply_all(q=q2)
        assert np.abs(v2[: dsc.nq] - 0.5 * np.array([1.0, -2.0, 0.5])).max() < 1e-11


def test_layer_targets_subset_matches_all():
    dsc = two_spheres(0.02, 6)
    rng = np.random.default_rng(7)
    f, q = rng.standard_normal((dsc.N, 3)), rng.standard_normal((dsc.N, 3))
    full = dsc.apply_all(f=f, q=q)
    tg = np.array([0, 5, dsc.nq + 3, dsc.N - 1])
    sub = dsc.apply(f=f, q=q, targets=tg)
    assert np.abs(sub - full[tg]).max() < 1e-13 * np.abs(full).max()


def test_single_sphere_mobility():
    for p in (6, 10):
        dsc = Disc(np.array([[0.3, 0.1, -2.0]]), p, a=1.3, mu=0.7)
        FT = np.array([[1.0, -2.0, 0.5, 0.3, 0.2, -0.7]])
        UO = mob.mobility(dsc, FT)
        assert np.abs(UO[0, :3] - FT[0, :3] / (6 * np.pi * 0.7 * 1.3)).max() < 1e-12
        assert np.abs(UO[0, 3:] - FT[0, 3:] / (8 * np.pi * 0.7 * 1.3 ** 3)).max() < 1e-12


def test_single_janus_sphere():
    """App. A.5: U = -<u_s> (quadrature mean), Omega = 0; -> (B/3) a as p grows."""
    ax = np.array([[0.3, -0.5, 0.81]])
    ax /= np.linalg.norm(ax)
    for p in (8, 12):
        dsc = Disc(np.zeros((1, 3)), p)
        us = mob.janus_slip(dsc, ax, B=1.0)
        UO = mob.mobility(dsc, np.zeros((1, 6)), us)
        # the discrete identity Pi_R A_op q = Pi_R q gives (U, Omega) = -Pi_R[u_s] exactly
        assert np.abs(UO[0] + mob.rigid_coeffs(dsc, us)[0]).max() < 1e-12
        assert np.abs(UO[0, 3:]).max() < 5e-2               # Omega -> 0 (quadrature of a jump)
    assert np.abs(UO[0, :3] - ax[0] / 3).max() < 2e-2   # discontinuous slip: slow convergence


def test_gmres_vs_dense_solve():
    dsc = two_spheres(0.1, 4)
    n = 3 * dsc.N
    A = np.stack([mob.A_op(dsc, e.reshape(-1, 3)).reshape(-1) for e in np.eye(n)], axis=1)
    rng = np.random.default_rng(9)
    rhs = rng.standard_normal(n)
    x, it, rr = mob.gmres(lambda v: mob.A_op(dsc, v.reshape(-1, 3)), rhs, tol=1e-14)
    xd = np.linalg.solve(A, rhs)
    assert np.abs(x - xd).max() < 1e-11 * np.abs(xd).max()


def test_rotation_covariance():
    """Rotating every centre by R_z(pi/p) permutes grid nodes: M' = R M R^T exactly."""
    p = 6
    C = np.array([[0.0, 0.0, 0.0], [2.3, 0.4, 0.2], [0.2, 2.1, 0.9]])
    R = rot_z(np.pi / p)
    FT = np.array([[1.0, 0.2, -0.3, 0.1, 0.0, 0.2], [0.0, -1.0, 0.5, 0.0, 0.3, 0.0], [0.3, 0.3, 0.3, -0.2, 0.1, 0.0]])
    d1 = Disc(C, p)
    d2 = Disc(C @ R.T, p)
    U1 = mob.mobility(d1, FT)
    FT2 = np.concatenate([FT[:, :3] @ R.T, FT[:, 3:] @ R.T], axis=1)
    U2 = mob.mobility(d2, FT2)
    U1r = np.concatenate([U1[:, :3] @ R.T, U1[:, 3:] @ R.T], axis=1)
    assert np.abs(U2 - U1r).max() < 1e-11 * np.abs(U1).max()


def test_far_spheres_rpy():
    d = 12.0
    dsc = Disc(np.array([[0.0, 0, 0], [d, 0, 0]]), 8)
    FT = np.zeros((2, 6))
    FT[1, :3] = [0.3, 1.0, -0.5]
    UO = mob.mobility(dsc, FT)
    rhat = np.array([1.0, 0, 0])
    a = 1.0
    M12 = ((1 + 2 * a * a / (3 * d * d)) * np.eye(3) + (1 - 2 * a * a / (d * d)) * np.outer(rhat, rhat)) / (8 * np.pi * d)
    ref = M12 @ FT[1, :3]
    assert np.abs(UO[0, :3] - ref).max() < 1e-4 * np.abs(ref).max()


def test_contacts_and_D():
    C = np.array([[0.0, 0, 0], [2.04, 0, 0], [4.2, 0.1, 0.0], [0.0, 2.08, 0.0]])
    pairs, nrm, gaps = lcp.contacts(C, 1.0, 0.1)
    assert [tuple(p) for p in pairs] == [(0, 1), (0, 3)]
    assert np.allclose(gaps, [0.04, 0.08])
    lam = np.array([0.7, 1.3])
    FT = lcp.D_apply(4, pairs, nrm, lam)
    # D column = finite difference of the gap w.r.t. centres: dPhi/dc_i = -n, dPhi/dc_j = +n
    for l, (i, j) in enumerate(pairs):
        for s, k in ((-1, i), (1, j)):
            for ax in range(3):
                Cp = C.copy()
                Cp[k, ax] += 1e-7
                gp = np.linalg.norm(Cp[j] - Cp[i]) - 2
                assert abs((gp - gaps[l]) / 1e-7 - s * nrm[l][ax]) < 1e-6
    assert np.allclose(FT[0, :3], -0.7 * nrm[0] - 1.3 * nrm[1])
    # D^T of a common translation is zero
    UO = np.tile([0.3, -0.2, 0.9, 0.1, 0.2, 0.3], (4, 1))
    assert np.abs(lcp.DT_apply(pairs, nrm, UO)).max() < 1e-15


def test_mobility_symmetric_pd():
    """P8 / R27: M symmetric to discretisation error (decreasing with p), PD."""
    C = np.array([[0.0, 0, 0], [2.3, 0.4, 0.1]])
    asyms = []
    for p in (4, 8):
        dsc = Disc(C, p)
        M = np.stack([mob.mobility(dsc, e.reshape(2, 6)).reshape(-1) for e in np.eye(12)], 1)
        asyms.append(np.abs(M - M.T).max() / np.abs(M).max())
        assert np.linalg.eigvalsh(0.5 * (M + M.T)).min() > 0
    assert asyms[1] < asyms[0] / 50 and asyms[1] < 1e-5, asyms


def test_lcp_matrix_pd_near_contact():
    """A = D^T M D positive definite on a 3-sphere contact scene (gaps 0.05-0.08)."""
    C = np.array([[0.0, 0, 0], [2.05, 0.1, 0], [1.0, 1.8, 0.05]])
    pairs, nrm, gaps = lcp.contacts(C, 1.0, 0.1)
    dsc = Disc(C, 5)
    A = lcp.densify(lambda v: lcp.lcp_mvp(dsc, pairs, nrm, v, tol=1e-13), len(pairs))
    assert np.linalg.eigvalsh(0.5 * (A + A.T)).min() > 0
    assert np.abs(A - A.T).max() / np.abs(A).max() < 0.1
