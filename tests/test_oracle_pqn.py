"""Pins for the oracle's PQN layer (not gpu): SPEC.md worked examples
(tests/golden/spec_examples.json), the weighted prox against a brute-force
active-set QP, eta* against a grid, CG equivalence on an interior QP
(PAPER.md P:289), sufficient decrease (App. B), MVP accounting
(P:356-358), and LCP solutions against brute-force enumeration."""
import itertools
import json
import os

import numpy as np
import pytest

from oracle import pqn
from oracle.lcp import brute_force_lcp

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def mvp_of(A):
    return lambda v: (A @ v, None)


def test_kkt_examples():
    for c in GOLD["kkt"][:2]:
        e, _ = pqn.kkt_errors(np.array(c["x"], float), np.array(c["grad"], float))
        assert abs(e - c["abs"]) < 1e-15
    c = GOLD["kkt"][2]
    _, rel = pqn.kkt_errors(np.array([c["abs_now"]]), np.array([c["abs_now"]]), c["abs_prev"])
    assert abs(rel - c["rel"]) < 1e-15


def test_weighted_prox_examples():
    for c in GOLD["weighted_prox"]:
        D = np.array(c["D"], float)
        U = np.array(c["U"], float).reshape(D.size, -1) if c["U"] else np.zeros((D.size, 0))
        V = np.array(c["V"], float).reshape(D.size, -1) if c["V"] else np.zeros((D.size, 0))
        z, _, _ = pqn.weighted_prox(D, U, V, np.array(c["xt"], float))
        assert np.abs(z - np.array(c["out"])).max() < 1e-12


def qp_brute(B, xt):
    """argmin_{z>=0} 1/2 (z-xt)^T B (z-xt) by enumerating the free set."""
    n = xt.size
    best, bestv = None, np.inf
    for mask in itertools.product([False, True], repeat=n):
        F = np.array(mask)
        z = np.zeros(n)
        if F.any():
            # stationarity on free set: B_FF (z_F - xt_F) - B_FA xt_A = 0
            A_ = ~F
            rhs = B[np.ix_(F, F)] @ xt[F] + B[np.ix_(F, A_)] @ xt[A_]
            z[F] = np.linalg.solve(B[np.ix_(F, F)], rhs)
        if (z < -1e-12).any():
            continue
        v = 0.5 * (z - xt) @ B @ (z - xt)
        if v < bestv:
            best, bestv = z, v
    return best


def test_weighted_prox_vs_dense_qp():
    """S:149 oracle suite: 500 random (D, U, V, x~) with B PD."""
    rng = np.random.default_rng(11)
    done = 0
    while done < 500:
        n = int(rng.integers(2, 8))
        r = int(rng.integers(1, 4))
        D = rng.uniform(0.5, 2.0, n)
        U = rng.standard_normal((n, r)) * 0.7
        V = rng.standard_normal((n, r)) * 0.4
        B = np.diag(D) + U @ U.T - V @ V.T
        if np.linalg.eigvalsh(B).min() < 0.05:
            continue
        xt = rng.standard_normal(n)
        z, it, res = pqn.weighted_prox(D, U, V, xt)
        ref = qp_brute(B, xt)
        assert np.abs(z - ref).max() < 1e-8, (n, r, z, ref)
        done += 1


def test_eta_examples_and_grid():
    for c in GOLD["optimal_eta"]:
        A = np.array(c["A"], float)
        b, x, p = (np.array(c[k], float) for k in ("b", "x", "p"))
        eta, _ = pqn.optimal_eta(x, p, A @ x + b, A @ p)
        assert abs(eta - c["eta"]) < 1e-14
    rng = np.random.default_rng(3)
    for _ in range(50):
        n = 6
        M = rng.standard_normal((n, n))
        A = M @ M.T + n * np.eye(n)
        b = rng.standard_normal(n)
        x = np.abs(rng.standard_normal(n)) * (rng.uniform(size=n) < 0.7)
        p = -(A @ x + b) * rng.uniform(0.5, 1.5, n)
        g = A @ x + b
        if p @ g >= 0:
            continue
        eta, _ = pqn.optimal_eta(x, p, g, A @ p)
        f = lambda e: 0.5 * (x + e * p) @ A @ (x + e * p) + b @ (x + e * p)
        neg = p < 0
        emax = (-x[neg] / p[neg]).min() if neg.any() else 10.0
        grid = np.linspace(0, emax, 10001)
        assert (x + eta * p >= -1e-15).all()
        assert f(eta) <= min(f(e) for e in grid) + 1e-10 * abs(f(0)) + 1e-14


def test_bfgs_examples_and_roundtrip():
    c = GOLD["bfgs"][0]
    q = pqn.BFGS(2)
    assert q.update(np.array(c["s"], float), np.array(c["y"], float))
    assert np.abs(q.B(np.array(c["s"], float)) - np.array(c["Bs"])).max() < 1e-15
    c = GOLD["bfgs"][1]
    assert np.abs(q.H(np.array(c["g"], float)) - np.array(c["Hg"])).max() < 1e-15
    rng = np.random.default_rng(4)
    n = 10
    M = rng.standard_normal((n, n))
    A = M @ M.T + np.eye(n)
    q = pqn.BFGS(n)
    for _ in range(3):
        s = rng.standard_normal(n)
        q.update(s, A @ s)
    for _ in range(5):
        x = rng.standard_normal(n)
        assert np.abs(q.H(q.B(x)) - x).max() < 1e-8 * np.abs(x).max()
    s = rng.standard_normal(n)
    q.update(s, A @ s)
    assert np.abs(q.B(s) - A @ s).max() < 1e-9 * np.abs(A @ s).max()    # latest secant exact
    assert pqn.BFGS(2).update(np.array([1.0, 0]), np.array([0.0, 1])) is False   # y^T s = 0 skip


def test_mono_pqn_examples():
    for c in GOLD["mono_pqn"]:
        A = np.array(c["A"], float)
        b = np.array(c["b"], float)
        x, g, _, _, rep = pqn.mono_pqn(mvp_of(A), b, np.zeros(2), eps_abs=1e-12)
        assert np.abs(x - np.array(c["x"])).max() < 1e-10
        assert rep["mvps"] == rep["iterations"] + 1
        if "mvps" in c:
            assert rep["mvps"] == c["mvps"]


def test_bi_pqn_identical_fidelity():
    c = GOLD["bi_pqn_identical_fidelity"]
    A = np.array(c["A"], float)
    b = np.array(c["b"], float)
    x, rep = pqn.bi_pqn(lambda v: A @ v, lambda v: A @ v, b, np.zeros(2), eps_abs=1e-12)
    assert rep["hi_mvps"] == c["hi_mvps"]
    assert np.abs(x - np.array([0.5, 0.0])).max() < 1e-10


def test_cg_equivalence():
    """on a QP whose iterates stay interior, PQN with exact line search = CG."""
    rng = np.random.default_rng(8)
    n = 8
    M = rng.standard_normal((n, n))
    A = M @ M.T + n * np.eye(n)
    xs = 10.0 + rng.uniform(size=n)
    b = -A @ xs
    x0 = xs + 0.1 * rng.standard_normal(n)
    x, g, _, _, rep = pqn.mono_pqn(mvp_of(A), b, x0, eps_abs=1e-13, k_max=n + 2)
    # plain CG from x0
    xc = x0.copy()
    r = -(A @ xc + b)
    d = r.copy()
    cg = [xc.copy()]
    for k in range(n):
        if np.linalg.norm(r) < 1e-13:
            break
        al = r @ r / (d @ A @ d)
        xc = xc + al * d
        rn = r - al * (A @ d)
        d = rn + (rn @ rn) / (r @ r) * d
        r = rn
        cg.append(xc.copy())
    for k in range(min(len(cg), len(rep["x_trace"]), 5)):
        assert np.abs(rep["x_trace"][k] - cg[k]).max() < 1e-8 * np.abs(xs).max(), k


@pytest.mark.parametrize("seed", range(6))
def test_lcp_solvers_vs_brute_force(seed):
    """P10: Mono-PQN, Bi-PQN (A^ = perturbed A) and brute force give the same
    unique LCP solution; sufficient decrease (App. B) holds on every step."""
    rng = np.random.default_rng(100 + seed)
    n = 9
    M = rng.standard_normal((n, n))
    A = M @ M.T / n + 0.3 * np.eye(n)
    b = rng.standard_normal(n)
    E = rng.standard_normal((n, n)) * 0.02
    Ahat = A + 0.5 * (E + E.T)
    ref, cnt = brute_force_lcp(A, b)
    assert cnt == 1
    x1, g1, _, _, r1 = pqn.mono_pqn(mvp_of(A), b, np.zeros(n), eps_abs=1e-12)
    assert r1["termination"] == pqn.TERM_KKT_ABS
    assert np.abs(x1 - ref).max() < 1e-9
    assert r1["mvps"] == r1["iterations"] + 1
    f = lambda x: 0.5 * x @ A @ x + b @ x
    xs = r1["x_trace"]
    for k in range(len(xs) - 1):
        p_dir = xs[k + 1] - xs[k]
        assert f(xs[k + 1]) <= f(xs[k]) + 0.25 * ((A @ xs[k] + b) @ p_dir) + 1e-14
    x2, r2 = pqn.bi_pqn(lambda v: A @ v, lambda v: Ahat @ v, b, np.zeros(n), eps_abs=1e-12)
    assert r2["termination"] == pqn.TERM_KKT_ABS
    assert np.abs(x2 - ref).max() < 1e-9
    assert r2["hi_mvps"] == r2["iterations"] + 1


# ------------------------------------------------------------------ BB-PGD (NEXT-1)
def test_bb_step_examples():
    """A = I -> 1; A = diag(2,1), s = (1,0) -> 0.5; random SPD -> in [1/l_max, 1/l_min]."""
    from oracle.pqn import bb_step
    s = np.array([0.3, -1.2])
    assert bb_step(s, s, 7.0) == pytest.approx(1.0, abs=1e-15)
    assert bb_step(np.array([1.0, 0.0]), np.array([2.0, 0.0]), 7.0) == pytest.approx(0.5, abs=1e-15)
    assert bb_step(np.array([1.0, -1.0]), np.array([-1.0, 1.0]), 7.0) == 7.0   # non-positive denominator
    rng = np.random.default_rng(4)
    M = rng.standard_normal((6, 6))
    A = M @ M.T + 0.1 * np.eye(6)
    ev = np.linalg.eigvalsh(A)
    for _ in range(20):
        s = rng.standard_normal(6)
        t = bb_step(s, A @ s, 0.0)
        assert 1 / ev[-1] - 1e-12 <= t <= 1 / ev[0] + 1e-12


def test_bb_pgd_examples():
    """A = I, b = (-1,-1), x0 = 0 -> (1,1) in one step; A = diag(1,10), b = (-1,-10) -> (1,1)."""
    from oracle.pqn import bb_pgd
    x, g, rep = bb_pgd(lambda v: v, np.array([-1.0, -1.0]), np.zeros(2))
    assert np.allclose(x, [1.0, 1.0], atol=1e-15) and rep["iterations"] == 1 and rep["mvps"] == 2
    A = np.diag([1.0, 10.0])
    x, g, rep = bb_pgd(lambda v: A @ v, np.array([-1.0, -10.0]), np.zeros(2), eps_abs=1e-8)
    assert np.allclose(x, [1.0, 1.0], atol=1e-8) and rep["kkt_abs"] <= 1e-8
    assert rep["mvps"] == rep["iterations"] + 1


@pytest.mark.parametrize("seed", range(4))
def test_bb_pgd_vs_brute_force(seed):
    from oracle.lcp import brute_force_lcp
    from oracle.pqn import bb_pgd
    rng = np.random.default_rng(50 + seed)
    n = 8
    M = rng.standard_normal((n, n))
    A = M @ M.T / n + 0.5 * np.eye(n)
    b = rng.standard_normal(n)
    x, g, rep = bb_pgd(lambda v: A @ v, b, np.zeros(n), eps_abs=1e-12, k_max=5000)
    ref, cnt = brute_force_lcp(A, b)
    assert cnt == 1 and rep["termination"] == 0
    np.testing.assert_allclose(x, ref, atol=1e-10)


def _model(Ahat, U, V):
    return Ahat + sum((np.outer(u, u) for u in U), np.zeros_like(Ahat)) - \
        sum((np.outer(v, v) for v in V), np.zeros_like(Ahat))


def test_secant_transform_dense_identity():
    """SPEC S:224-229 / PAPER P:475-487 (reading R34): pairs with B^(k) S = Y become pairs of
    B^(k+1) = B^(k) + uu^T - vv^T; checked with dense matrices (n = 6, m = 2 and larger)."""
    assert pqn.transform_secants([], [], np.ones(3), np.ones(3)) == []            # empty cache
    s0, y0 = np.arange(3.0), np.arange(3.0) + 1
    y1 = pqn.transform_secants([s0], [y0], np.zeros(3), np.zeros(3))[0]           # u = v = 0
    assert np.array_equal(y1, y0)
    rng = np.random.default_rng(229)
    for n, m in [(6, 2), (12, 5), (40, 9)]:
        M = rng.standard_normal((n, n))
        Ahat = M @ M.T + np.eye(n)
        U = [rng.standard_normal(n) for _ in range(2)]
        V = [0.3 * rng.standard_normal(n) for _ in range(2)]
        Bk = _model(Ahat, U, V)
        S = [rng.standard_normal(n) for _ in range(m)]
        Y = [Bk @ s for s in S]
        u, v = rng.standard_normal(n), 0.5 * rng.standard_normal(n)
        Bk1 = Bk + np.outer(u, u) - np.outer(v, v)
        Yn = pqn.transform_secants(S, Y, u, v)
        for s, y in zip(S, Yn):
            assert np.abs(Bk1 @ s - y).max() <= 1e-12 * max(1.0, np.abs(y).max())
        # the display printed at P:486 / P:509 ("Y^ - (uu^T - vv^T) S^") breaks the identity
        Yp = [y - u * (u @ s) + v * (v @ s) for s, y in zip(S, Y)]
        assert max(np.abs(Bk1 @ s - y).max() for s, y in zip(S, Yp)) > 1e-3


def _bifi_lcp(seed, n):
    rng = np.random.default_rng(seed)
    M = rng.standard_normal((n, n))
    A = M @ M.T / n + 0.2 * np.eye(n)
    E = rng.standard_normal((n, n)) * 0.15 / np.sqrt(n)
    Ahat = A + E + E.T
    Ahat += max(0.0, 0.05 - np.linalg.eigvalsh(Ahat).min()) * np.eye(n)
    return A, Ahat, rng.standard_normal(n)


@pytest.mark.parametrize("seed", range(4))
def test_bi_pqn_reused_secants_fit_current_model(seed):
    """Inside Alg. 3 every seeded subproblem pair satisfies B^(k) s = y -- the
    property the secant re-use exists for -- and the solution is the unique LCP solution."""
    A, Ahat, b = _bifi_lcp(300 + seed, 24)
    x, rep = pqn.bi_pqn(lambda v: A @ v, lambda v: Ahat @ v, b, np.zeros(b.size), eps_abs=1e-11,
                        verify_secants=True)
    assert rep["termination"] == pqn.TERM_KKT_ABS
    assert len(rep["secant_residuals"]) >= 2
    assert max(rep["secant_residuals"]) <= 1e-10, rep["secant_residuals"]
    xm, _, _, _, _ = pqn.mono_pqn(mvp_of(A), b, np.zeros(b.size), eps_abs=1e-12)
    np.testing.assert_allclose(x, xm, atol=1e-9)
