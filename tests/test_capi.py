"""C-ABI boundary checks that need no GPU.

* libbpqn.so builds for sm_100a, loads, and exports every symbol include/bpqn.h declares;
* the Python binding marshals exactly those names;
* the host-side PQN solvers behind bpqn_solve_lcp_dense (no device work) reproduce
  SPEC.md's worked examples (tests/golden/spec_examples.json) and the brute-force
  LCP solution of random small P-matrix LCPs.
"""
import json
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2604_10089_b200 import build as b
    b.build()
    import paper_2604_10089_b200 as bp
    return bp.lib()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "bpqn.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bpqn_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_boundary():
    syms = header_symbols()
    for name in ["bpqn_geometry_init", "bpqn_contacts", "bpqn_mobility_apply", "bpqn_lcp_mvp", "bpqn_solve_lcp"]:
        assert name in syms   # BASELINE.json north_star's export list


def test_library_exports_every_declared_symbol(lib):
    so = os.path.join(ROOT, "paper_2604_10089_b200", "libbpqn.so")
    out = subprocess.check_output(["nm", "-D", "--defined-only", so]).decode()
    exported = set(re.findall(r"\bT (bpqn_[a-z0-9_]+)", out))
    missing = [s for s in header_symbols() if s not in exported]
    assert not missing, missing
    for s in header_symbols():
        getattr(lib, s)


def test_binding_covers_header():
    from paper_2604_10089_b200 import _bpqn
    assert sorted(_bpqn.SYMBOLS) == header_symbols()


def test_sm100a_code_in_library(lib):
    so = os.path.join(ROOT, "paper_2604_10089_b200", "libbpqn.so")
    out = subprocess.check_output(["cuobjdump", "--list-elf", so]).decode()
    assert "sm_100a" in out


def test_no_device_errors_are_loud(lib):
    """Without a usable device a compute call fails with BPQN_ERR_CUDA, never silently."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2604_10089_b200 as bp
    with pytest.raises(bp.BpqnError) as e:
        bp.Geometry(np.zeros((1, 3)), 4, stream=0)
    assert e.value.code == 2


def _golden():
    with open(os.path.join(ROOT, "tests", "golden", "spec_examples.json")) as fh:
        return json.load(fh)


def test_dense_mono_pqn_spec_example(lib):
    """mono_pqn on A = [[2,0],[0,1]], b = (-1, 1) -> x = (0.5, 0)."""
    import paper_2604_10089_b200 as bp
    A = np.array([[2.0, 0.0], [0.0, 1.0]])
    b = np.array([-1.0, 1.0])
    x, rep, rc = bp.solve_lcp_dense(A, b)
    assert rc == 0
    np.testing.assert_allclose(x, [0.5, 0.0], atol=1e-12)
    assert rep.hi_mvps == rep.iterations + 1 + rep.iterations // 20   # 1/iteration + initial + refresh (R18)


def test_dense_bi_pqn_identical_fidelity(lib):
    """Bi-PQN with A_hat == A converges with a single hi MVP after the lo init."""
    import paper_2604_10089_b200 as bp
    rng = np.random.default_rng(3)
    M = rng.standard_normal((6, 6))
    A = M @ M.T + 6 * np.eye(6)
    b = rng.standard_normal(6)
    o = bp.default_solve_opts(method=1, eps_kkt_abs=1e-11)
    x, rep, rc = bp.solve_lcp_dense(A, b, Ahat=A, opts=o)
    assert rc == 0
    assert rep.hi_mvps == 1
    w = A @ x + b
    assert np.linalg.norm(np.minimum(x, w)) <= 1e-10


def _brute(A, b):
    import itertools
    n = b.size
    for mask in itertools.product([False, True], repeat=n):
        S = np.array(mask)
        lam = np.zeros(n)
        if S.any():
            lam[S] = np.linalg.solve(A[np.ix_(S, S)], -b[S])
        if (lam < -1e-12).any():
            continue
        if ((A @ lam + b)[~S] < -1e-12).any():
            continue
        return lam
    return None


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("method", [0, 1])
def test_dense_pqn_vs_brute_force(lib, seed, method):
    """Host PQN (C++) on random SPD LCPs of size 7 equals active-set enumeration (O14)."""
    import paper_2604_10089_b200 as bp
    rng = np.random.default_rng(100 + seed)
    n = 7
    M = rng.standard_normal((n, n))
    A = M @ M.T + 0.5 * np.eye(n)
    b = rng.standard_normal(n)
    Ahat = A + 0.05 * (lambda E: E + E.T)(rng.standard_normal((n, n))) if method == 1 else None
    if Ahat is not None:
        Ahat = Ahat + n * 0.1 * np.eye(n)
    o = bp.default_solve_opts(method=method, eps_kkt_abs=1e-12)
    x, rep, rc = bp.solve_lcp_dense(A, b, Ahat=Ahat, opts=o)
    assert rc == 0, rep.as_dict()
    ref = _brute(A, b)
    np.testing.assert_allclose(x, ref, atol=1e-9)
    if method == 1:
        assert rep.hi_mvps == rep.iterations + 1 + rep.iterations // 20  # P:574 + refresh every 20 (R18)


@pytest.mark.parametrize("seed", range(4))
def test_dense_bb_pgd_vs_brute_force(lib, seed):
    """BB-PGD (method 2) behind the C ABI: SPEC S:366-367 and brute-force LCPs."""
    import paper_2604_10089_b200 as bp
    o = bp.default_solve_opts(method=2, eps_kkt_abs=1e-12, k_max=5000)
    x, rep, rc = bp.solve_lcp_dense(np.eye(2), np.array([-1.0, -1.0]), opts=o)
    assert rc == 0 and rep.iterations == 1 and np.allclose(x, [1.0, 1.0])
    rng = np.random.default_rng(50 + seed)
    n = 8
    M = rng.standard_normal((n, n))
    A = M @ M.T / n + 0.5 * np.eye(n)
    b = rng.standard_normal(n)
    x, rep, rc = bp.solve_lcp_dense(A, b, opts=o)
    assert rc == 0
    np.testing.assert_allclose(x, _brute(A, b), atol=1e-10)
    assert rep.hi_mvps == rep.iterations + 1


@pytest.mark.parametrize("seed", range(3))
def test_dense_bi_pqn_secant_reuse(lib, seed):
    """C++ Bi-PQN behind the C ABI: every re-used subproblem secant pair fits the current model
    B^(k) s = y (reading R34), and the LCP solution is unchanged."""
    import paper_2604_10089_b200 as bp
    rng = np.random.default_rng(300 + seed)
    n = 24
    M = rng.standard_normal((n, n))
    A = M @ M.T / n + 0.2 * np.eye(n)
    E = rng.standard_normal((n, n)) * 0.15 / np.sqrt(n)
    Ahat = A + E + E.T
    Ahat += max(0.0, 0.05 - np.linalg.eigvalsh(Ahat).min()) * np.eye(n)
    b = rng.standard_normal(n)
    o = bp.default_solve_opts(method=1, eps_kkt_abs=1e-11, verify_secants=1)
    x, rep, rc = bp.solve_lcp_dense(A, b, Ahat=Ahat, opts=o)
    assert rc == 0
    assert 0 < rep.secant_residual <= 1e-10, rep.secant_residual
    xm, _, _ = bp.solve_lcp_dense(A, b, opts=bp.default_solve_opts(method=0, eps_kkt_abs=1e-12))
    np.testing.assert_allclose(x, xm, atol=1e-9)


def test_c4_certificate():
    """The oracle's KKT certificate of the c4 LCP solution (R26 / DESIGN.md R35): the stored
    A_oracle lambda_cert (one oracle MVP, tests/fixtures/make_fixtures.py --certify 4) and the
    oracle's b give ||min(lambda, A lambda + b)||_2 <= 1e-8; recomputed here from the stored oracle
    values (lambda_cert >= 0, complementarity on the active set, dual feasibility off it)."""
    import os
    path = os.path.join(os.path.dirname(__file__), "fixtures", "c4.npz")
    z = np.load(path, allow_pickle=True)
    if "lam_cert" not in z:
        pytest.skip("c4 certificate not generated")
    lam, w, b = z["lam_cert"], z["A_lam_cert"], z["b"]
    assert (lam >= 0).all()
    kkt = np.linalg.norm(np.minimum(lam, w + b))
    assert abs(kkt - float(z["cert_kkt"])) <= 1e-15 + 1e-12 * kkt
    assert kkt <= 1e-8
    g = w + b
    assert (g[lam == 0] >= -1e-8).all() and np.abs(g[lam > 1e-12]).max() <= 1e-8
