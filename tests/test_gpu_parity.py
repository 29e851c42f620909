"""GPU parity: the CUDA path (libbpqn through the C ABI) against the CPU oracle.

Tolerances (BASELINE.json north_star): fp64 relative L2
  <= 1e-11  one kernel summation (bpqn_layer_apply),
  <= 1e-9   GMRES-solved velocities (mobility, LCP MVP, b),
  <= 1e-7   lambda of the LCP solve, complementarity residual <= 1e-8 evaluated
            with the ORACLE's operator on the GPU's lambda (R26);
bit-exact for the contact index set.
Small scenes are computed by the oracle on the fly; c1-c4 operator/LCP outputs
come from tests/fixtures/c*.npz written by tests/fixtures/make_fixtures.py,
which calls only oracle/.  Full-size c4/c5 layer applies are checked on sampled
targets the oracle computes one by one.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIX = os.path.join(ROOT, "tests", "fixtures")

TOL_SUM, TOL_VEL, TOL_LAM, TOL_KKT = 1e-11, 1e-9, 1e-7, 1e-8
GM_PARITY = dict(tol=1e-12)


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def bp():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2604_10089_b200 as m
    m.lib()
    return m


def T(x, dtype=None):
    import torch
    return torch.tensor(np.asarray(x), dtype=dtype or torch.float64, device="cuda")


def fixture(c):
    path = os.path.join(FIX, "c%d.npz" % c)
    if not os.path.exists(path):
        pytest.skip("fixture c%d.npz not generated" % c)
    return np.load(path, allow_pickle=True)


SCENES = {
    "two_near_p6": (np.array([[0.1, -0.2, 0.3], [2.15, 0.4, 0.1]]), 6),
    "three_p5": (np.array([[0.0, 0.0, 0.0], [2.05, 0.1, 0.0], [1.025, 1.9, 0.05]]), 5),
    "touching_gap_1e-3_p8": (np.array([[0.0, 0.0, 0.0], 2.001 * np.array([0.3, 0.8, 0.6]) / np.sqrt(1.09)]), 8),
    "single_p2": (np.array([[0.3, 0.2, -0.1]]), 2),
    "single_p7": (np.array([[0.0, 0.0, 0.0]]), 7),
}


def _scene(name):
    return SCENES[name]


# ------------------------------------------------------------------ layer operator (K1 + K2 + K3)
@pytest.mark.parametrize("name", list(SCENES))
def test_layer_apply_small(bp, name):
    from oracle.layer import Disc
    C, p = _scene(name)
    d = Disc(C, p)
    g = bp.Geometry(C, p)
    assert g.N == d.N and g.n_incidences == len(d.inc)
    rng = np.random.default_rng(11)
    f, q = rng.standard_normal((d.N, 3)), rng.standard_normal((d.N, 3))
    ref_s, ref_d = d.apply_all(f=f), d.apply_all(q=q)
    us = bp.layer_apply(g, f=T(f)).cpu().numpy()
    ud = bp.layer_apply(g, q=T(q)).cpu().numpy()
    usd = bp.layer_apply(g, f=T(f), q=T(q)).cpu().numpy()
    assert rel(us, ref_s) <= TOL_SUM
    assert rel(ud, ref_d) <= TOL_SUM
    assert rel(usd, ref_s + ref_d) <= TOL_SUM


@pytest.mark.parametrize("a,mu", [(0.7, 1.3), (2.5, 0.4)])
def test_layer_apply_radius_viscosity(bp, a, mu):
    """Spheres of radius a != 1 in a fluid of viscosity mu != 1 (the near rule's graded theta' panel,
    the rotation-form tensors and the self rules all scale with a): three spheres at gaps 0.004 a /
    0.05 a against the oracle."""
    from oracle.layer import Disc
    e = np.array([0.6, -0.48, 0.64])
    C = np.array([[0.2, 0.1, -0.3], [0.2, 0.1, -0.3] + a * 2.004 * e,
                  [0.2, 0.1, -0.3] + a * np.array([0.3, 2.05, 0.1]) / np.linalg.norm([0.3, 2.05, 0.1]) * 2.05])
    p = 7
    d = Disc(C, p, a, mu)
    g = bp.Geometry(C, p, radius=a, mu=mu)
    assert g.N == d.N and g.n_incidences == len(d.inc) > 0
    rng = np.random.default_rng(13)
    f, q = rng.standard_normal((d.N, 3)), rng.standard_normal((d.N, 3))
    usd = bp.layer_apply(g, f=T(f), q=T(q)).cpu().numpy()
    assert rel(usd, d.apply_all(f=f) + d.apply_all(q=q)) <= TOL_SUM


def _random_scene(seed):
    """Seeded random packing: 2-12 unit spheres, gaps >= 0.01, order p in 3..9 (both K1 variants,
    ragged target blocks and source tiles, near and far pairs)."""
    rng = np.random.default_rng(1000 + seed)
    np_, p = int(rng.integers(2, 13)), int(rng.integers(3, 10))
    C = []
    while len(C) < np_:
        c = rng.uniform(0.0, 2.6 * np_ ** (1 / 3) + 1.0, 3)
        if all(np.linalg.norm(c - o) >= 2.01 for o in C):
            C.append(c)
    return np.array(C), p


@pytest.mark.parametrize("seed", range(8))
def test_layer_apply_random_scenes(bp, seed):
    """All targets of seeded random scenes (every mode) against the oracle's full apply."""
    from oracle.layer import Disc
    C, p = _random_scene(seed)
    d = Disc(C, p)
    g = bp.Geometry(C, p)
    assert g.N == d.N and g.n_incidences == len(d.inc)
    rng = np.random.default_rng(seed)
    f, q = rng.standard_normal((d.N, 3)), rng.standard_normal((d.N, 3))
    ref_s, ref_d = d.apply_all(f=f), d.apply_all(q=q)
    usd = bp.layer_apply(g, f=T(f), q=T(q)).cpu().numpy()
    ud = bp.layer_apply(g, q=T(q)).cpu().numpy()
    us = bp.layer_apply(g, f=T(f)).cpu().numpy()
    assert rel(us, ref_s) <= TOL_SUM, (C.shape[0], p)
    assert rel(ud, ref_d) <= TOL_SUM, (C.shape[0], p)
    assert rel(usd, ref_s + ref_d) <= TOL_SUM, (C.shape[0], p)


def test_layer_apply_none_is_zero(bp):
    C, p = _scene("three_p5")
    g = bp.Geometry(C, p)
    u = bp.layer_apply(g).cpu().numpy()
    assert not u.any()


def _sample_targets(d, n, seed):
    rng = np.random.default_rng(seed)
    t = set(rng.choice(d.N, size=n, replace=False).tolist())
    t.update([0, d.N - 1, d.nq - 1, d.nq])                      # ends and a sphere boundary
    if len(d.inc):
        t.update(np.unique(d.inc_t)[rng.choice(len(np.unique(d.inc_t)), size=min(n, 16), replace=False)].tolist())
    return np.array(sorted(t), dtype=np.int64)


@pytest.mark.parametrize("c", [1, 2, 3, 4, 5])
def test_layer_apply_config_sampled(bp, c):
    """Full-size layer apply (the launch configuration bench.py times) on sampled
    targets: random, sphere boundaries and near-incidence targets."""
    from oracle.layer import Disc
    from synth import layer_densities, make_config
    cfg = make_config(c)
    d = Disc(cfg["centers"], cfg["p"], cfg["radius"], cfg["mu"])
    g = bp.Geometry(cfg["centers"], cfg["p"], cfg["radius"], cfg["mu"])
    assert g.N == d.N and g.n_incidences == len(d.inc)
    f, q = layer_densities(c, d.N)
    u = bp.layer_apply(g, f=T(f), q=T(q)).cpu().numpy()
    tg = _sample_targets(d, 24 if c >= 4 else 48, 100 + c)
    ref = d.apply(f=f, q=q, targets=tg)
    assert rel(u[tg], ref) <= TOL_SUM, rel(u[tg], ref)
    assert np.isfinite(u).all()


def test_layer_apply_block_padding_regression(bp):
    """118 spheres at p = 16: N = 64 192 lies just above a multiple of the symmetric K1's
    1280-point target block but below the next 9216 -- the packed records must cover the
    last block for every launch shape.  An S+D apply first leaves 80-byte records in the
    buffer; the D and S applies that follow must not read them as sources."""
    from oracle.layer import Disc
    rng = np.random.default_rng(7)
    g1 = np.arange(5) * 2.05
    C = np.array([[x, y, z] for x in g1 for y in g1 for z in g1])[:118] + rng.uniform(-0.01, 0.01, (118, 3))
    d = Disc(C, 16)
    g = bp.Geometry(C, 16)
    assert g.N == 64192
    f, q = rng.standard_normal((g.N, 3)), rng.standard_normal((g.N, 3))
    bp.layer_apply(g, f=T(f), q=T(q))
    tg = _sample_targets(d, 24, 7)
    ud = bp.layer_apply(g, q=T(q)).cpu().numpy()
    assert rel(ud[tg], d.apply(q=q, targets=tg)) <= TOL_SUM
    us = bp.layer_apply(g, f=T(f)).cpu().numpy()
    assert rel(us[tg], d.apply(f=f, targets=tg)) <= TOL_SUM


@pytest.mark.parametrize("nsph,p", [(70, 12), (41, 16), (125, 3)])
def test_layer_apply_ragged_blocks(bp, nsph, p):
    """Mid-size scenes whose N is not a multiple of the K1 target block (70 x 312 = 21 840
    with 1024-point blocks; 41 x 544 = 22 304), sampled targets against the oracle; 125 spheres at
    p = 3 (Nq = 24 < 32: the one-directional K1 over three 1024-row blocks and its segment partials)."""
    from oracle.layer import Disc
    rng = np.random.default_rng(nsph)
    g1 = np.arange(5) * 2.04
    C = np.array([[x, y, z] for x in g1 for y in g1 for z in g1])[:nsph] + rng.uniform(-0.01, 0.01, (nsph, 3))
    d = Disc(C, p)
    g = bp.Geometry(C, p)
    f, q = rng.standard_normal((g.N, 3)), rng.standard_normal((g.N, 3))
    u = bp.layer_apply(g, f=T(f), q=T(q)).cpu().numpy()
    tg = _sample_targets(d, 24, nsph)
    assert rel(u[tg], d.apply(f=f, q=q, targets=tg)) <= TOL_SUM
    ud = bp.layer_apply(g, q=T(q)).cpu().numpy()
    assert rel(ud[tg], d.apply(q=q, targets=tg)) <= TOL_SUM


# ------------------------------------------------------------------ mobility (K4 GMRES)
@pytest.mark.parametrize("name", ["two_near_p6", "three_p5", "single_p7"])
def test_mobility_small(bp, name):
    from oracle import mobility as mob
    from oracle.layer import Disc
    C, p = _scene(name)
    d = Disc(C, p)
    g = bp.Geometry(C, p)
    FT = np.random.default_rng(5).standard_normal((len(C), 6))
    uo, st = bp.mobility_apply(g, T(FT), gmres=bp.default_gmres_opts(**GM_PARITY))
    ref = mob.mobility(d, FT, tol=1e-13)
    assert rel(uo.cpu().numpy(), ref) <= TOL_VEL
    assert st.rel_resid <= 1e-12


@pytest.mark.parametrize("p", [10, 25])
def test_mobility_single_sphere_stokes_drag(bp, p):
    """GPU path against the closed form U = F/(6 pi mu a), Omega = T/(8 pi mu a^3) (App. A.1);
    p = 25 is the largest supported order (the precompute's full tile capacity)."""
    a, mu = 1.3, 0.7
    g = bp.Geometry(np.array([[1.0, -2.0, 0.5]]), p, radius=a, mu=mu)
    FT = np.array([[0.3, -1.2, 0.8, 0.5, 0.1, -0.7]])
    uo, _ = bp.mobility_apply(g, T(FT), gmres=bp.default_gmres_opts(**GM_PARITY))
    uo = uo.cpu().numpy()[0]
    np.testing.assert_allclose(uo[:3], FT[0, :3] / (6 * np.pi * mu * a), rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(uo[3:], FT[0, 3:] / (8 * np.pi * mu * a ** 3), rtol=1e-10, atol=1e-12)


def test_janus_slip_and_swim_speed(bp):
    from oracle import mobility as mob
    from oracle.layer import Disc
    C = np.array([[0.0, 0.0, 0.0], [3.0, 0.5, 0.0]])
    axes = np.array([[0.0, 0.0, 1.0], [0.6, 0.0, 0.8]])
    d = Disc(C, 8)
    g = bp.Geometry(C, 8)
    s = bp.janus_slip(g, axes, 1.0).cpu().numpy()
    np.testing.assert_allclose(s, mob.janus_slip(d, axes, 1.0), atol=1e-15)
    uo, _ = bp.mobility_apply(g, T(np.zeros((2, 6))), slip=T(s), gmres=bp.default_gmres_opts(**GM_PARITY))
    ref = mob.mobility(d, np.zeros((2, 6)), slip=s, tol=1e-13)
    assert rel(uo.cpu().numpy(), ref) <= TOL_VEL


@pytest.mark.parametrize("c", [1, 2, 3])
def test_mobility_config(bp, c):
    z = fixture(c)
    g = bp.Geometry(z["centers"], int(z["p"]))
    uo, st = bp.mobility_apply(g, T(z["FT_test"]), gmres=bp.default_gmres_opts(**GM_PARITY))
    assert rel(uo.cpu().numpy(), z["UO_test"]) <= TOL_VEL


# ------------------------------------------------------------------ contacts (K5)
@pytest.mark.parametrize("c", [1, 2, 3, 4, 5])
def test_contacts_bit_exact(bp, c):
    from oracle import lcp
    from synth import make_config
    cfg = make_config(c)
    g = bp.Geometry(cfg["centers"], 2)
    pairs, nrm, gaps = bp.contacts(g, cfg["delta"])
    op, on, og = lcp.contacts(cfg["centers"], cfg["radius"], cfg["delta"])
    assert np.array_equal(pairs.cpu().numpy().astype(np.int64), op)
    np.testing.assert_allclose(nrm.cpu().numpy(), on, atol=1e-15)
    np.testing.assert_allclose(gaps.cpu().numpy(), og, atol=1e-14)


def test_contacts_edge_cases(bp):
    import torch
    C = np.array([[0.0, 0.0, 0.0], [2.05, 0.0, 0.0], [4.1, 0.0, 0.0], [20.0, 0.0, 0.0]])
    g = bp.Geometry(C, 3)
    p, n, gp = bp.contacts(g, 0.0)            # no pair has gap < 0
    assert p.shape[0] == 0 and g.nc == 0
    with pytest.raises(bp.BpqnError):         # MVP with an empty contact set is an input error
        bp.lcp_mvp(g, torch.zeros(1, dtype=torch.float64, device="cuda"))
    with pytest.raises(bp.BpqnError) as e:    # capacity: 2 contacts, room for 1
        bp.contacts(g, 0.1, max_contacts=1)
    assert e.value.code == 7
    p, n, gp = bp.contacts(g, 0.1)
    assert p.cpu().numpy().tolist() == [[0, 1], [1, 2]]


def test_overlap_and_bad_args_rejected(bp):
    with pytest.raises(bp.BpqnError) as e:
        bp.Geometry(np.array([[0.0, 0.0, 0.0], [1.99, 0.0, 0.0]]), 4)
    assert e.value.code == 1
    with pytest.raises(bp.BpqnError) as e:
        bp.Geometry(np.array([[0.0, 0.0, 0.0]]), 1)
    assert e.value.code == 1
    with pytest.raises(bp.BpqnError) as e:          # beyond the precompute's tile capacity
        bp.Geometry(np.array([[0.0, 0.0, 0.0]]), 26)
    assert e.value.code == 1
    bp.Geometry(np.array([[0.0, 0.0, 0.0]]), 25)    # the largest supported order builds


def test_nan_input_reported(bp):
    C, p = _scene("two_near_p6")
    g = bp.Geometry(C, p)
    FT = np.zeros((2, 6))
    FT[0, 0] = np.nan
    with pytest.raises(bp.BpqnError) as e:
        bp.mobility_apply(g, T(FT))
    assert e.value.code == 6


# ------------------------------------------------------------------ LCP MVP and b
@pytest.mark.parametrize("c", [1, 2, 3, 4])
def test_lcp_mvp_config(bp, c):
    import torch
    z = fixture(c)
    g = bp.Geometry(z["centers"], int(z["p"]))
    pairs, nrm, gaps = bp.contacts(g, 0.1)
    assert np.array_equal(pairs.cpu().numpy().astype(np.int64), z["pairs"])
    for k in range(z["w_test"].shape[0]):
        from synth import lambda_test
        lam = lambda_test(c, g.nc, k)
        w, st = bp.lcp_mvp(g, T(lam), gmres=bp.default_gmres_opts(**GM_PARITY))
        assert rel(w.cpu().numpy(), z["w_test"][k]) <= TOL_VEL, (k, st.iters)
    del torch


@pytest.mark.parametrize("c", [1, 2, 3, 4])
def test_lcp_b_config(bp, c):
    from synth import make_config
    z = fixture(c)
    cfg = make_config(c)
    g = bp.Geometry(z["centers"], int(z["p"]))
    bp.contacts(g, 0.1)
    slip = bp.janus_slip(g, cfg["axes"], cfg["slip_B"])
    b, _ = bp.lcp_b(g, T(cfg["F_nc"]), slip=slip, gmres=bp.default_gmres_opts(**GM_PARITY))
    assert rel(b.cpu().numpy(), z["b"]) <= TOL_VEL


def test_lcp_mvp_unit_vectors_c1(bp):
    """Every column of A = D^T M D at c1 against the oracle's densified A."""
    z = fixture(1)
    g = bp.Geometry(z["centers"], int(z["p"]))
    bp.contacts(g, 0.1)
    A = z["A_dense"]
    for l in range(g.nc):
        e = np.zeros(g.nc)
        e[l] = 1.0
        w, _ = bp.lcp_mvp(g, T(e), gmres=bp.default_gmres_opts(**GM_PARITY))
        assert rel(w.cpu().numpy(), A[:, l]) <= TOL_VEL


# ------------------------------------------------------------------ LCP solves (host PQN over device MVPs)
def _kkt(lam, A, b):
    return float(np.linalg.norm(np.minimum(lam, A @ lam + b)))


def test_solve_lcp_mono_c1(bp):
    z = fixture(1)
    g = bp.Geometry(z["centers"], int(z["p"]))
    bp.contacts(g, 0.1)
    o = bp.default_solve_opts(method=0, eps_kkt_abs=1e-10)
    o.gm_hi.tol = 1e-12
    lam = T(np.zeros(g.nc))
    lam, rep, rc = bp.solve_lcp(g, None, T(z["b"]), lam, opts=o)
    assert rc == 0
    x = lam.cpu().numpy()
    assert rel(x, z["lam_brute"]) <= TOL_LAM
    assert _kkt(x, z["A_dense"], z["b"]) <= TOL_KKT
    assert rep.hi_mvps == rep.iterations + 1 + rep.iterations // 20  # P:574 + refresh every 20 (R18)


@pytest.mark.parametrize("method", ["mono", "bi"])
def test_solve_lcp_c2(bp, method):
    z = fixture(2)
    key = "lam_" + method
    if key not in z:
        pytest.skip("no %s solution in fixture" % method)
    g = bp.Geometry(z["centers"], int(z["p"]))
    bp.contacts(g, 0.1)
    lo = None
    if method == "bi":
        lo = bp.Geometry(z["centers"], int(z["p_lo"]))
        pr, nr, gp = bp.contacts(g, 0.1)
        bp.set_contacts(lo, pr, nr, gp)
    o = bp.default_solve_opts(method=1 if method == "bi" else 0, eps_kkt_abs=1e-10)
    o.gm_hi.tol = 1e-12
    o.gm_lo.tol = 1e-12
    lam = T(np.zeros(g.nc))
    lam, rep, rc = bp.solve_lcp(g, lo, T(z["b"]), lam, opts=o)
    assert rc == 0
    assert rel(lam.cpu().numpy(), z[key]) <= TOL_LAM
    if "A_dense" not in z:
        pytest.skip("c2 fixture lacks the oracle's densified A (make_fixtures.py --dense 2)")
    assert _kkt(lam.cpu().numpy(), z["A_dense"], z["b"]) <= TOL_KKT    # R26: the ORACLE's A on the GPU's lambda
    assert rep.hi_mvps == rep.iterations + 1 + rep.iterations // 20  # P:574 + refresh every 20 (R18)


def test_solve_lcp_bi_c3(bp):
    z = fixture(3)
    if "lam_bi" not in z:
        pytest.skip("no bi solution in fixture")
    g = bp.Geometry(z["centers"], int(z["p"]))
    pr, nr, gp = bp.contacts(g, 0.1)
    lo = bp.Geometry(z["centers"], int(z["p_lo"]))
    bp.set_contacts(lo, pr, nr, gp)
    o = bp.default_solve_opts(method=1, eps_kkt_abs=1e-10)
    o.gm_hi.tol = 1e-12
    o.gm_lo.tol = 1e-12
    lam, rep, rc = bp.solve_lcp(g, lo, T(z["b"]), T(np.zeros(g.nc)), opts=o)
    assert rc == 0
    assert rel(lam.cpu().numpy(), z["lam_bi"]) <= TOL_LAM
    if "A_dense" not in z:
        pytest.skip("c3 fixture lacks the oracle's densified A (make_fixtures.py --dense 3)")
    assert _kkt(lam.cpu().numpy(), z["A_dense"], z["b"]) <= TOL_KKT    # R26: the ORACLE's A on the GPU's lambda


def test_solve_lcp_bi_c4_certified(bp):
    """c4, the north-star config: a full Bi-PQN solve (Alg. 3, low fidelity p = 8) at parity settings
    (GMRES 1e-12, KKT 1e-10) equals the certified solution lambda_cert to 1e-7 (R35).  lambda_cert's
    certificate is the ORACLE's: ||min(lambda_cert, A_oracle lambda_cert + b_oracle)|| (one oracle MVP,
    tests/fixtures/make_fixtures.py --certify 4), pinned on the CPU by
    test_capi.py::test_c4_certificate; A is positive definite (Lemma 2), so a small
    oracle KKT residual bounds the distance to the oracle's unique solution."""
    z = fixture(4)
    if "lam_cert" not in z:
        pytest.skip("c4 fixture has no certificate yet")
    assert z["cert_kkt"] <= TOL_KKT
    from synth import make_config
    cfg = make_config(4)
    g = bp.Geometry(z["centers"], int(z["p"]))
    pr, nr, gp = bp.contacts(g, 0.1)
    assert np.array_equal(pr.cpu().numpy(), z["pairs"])
    lo = bp.Geometry(z["centers"], cfg["p_lo"])
    bp.set_contacts(lo, pr, nr, gp)
    gm = bp.default_gmres_opts(tol=1e-12)
    slip = bp.janus_slip(g, cfg["axes"], cfg["slip_B"])
    b, _ = bp.lcp_b(g, T(cfg["F_nc"]), slip=slip, gmres=gm)
    assert rel(b.cpu().numpy(), z["b"]) <= TOL_VEL
    o = bp.default_solve_opts(method=1, eps_kkt_abs=1e-10)
    o.gm_hi.tol = 1e-12
    o.gm_lo.tol = 1e-12
    lam, rep, rc = bp.solve_lcp(g, lo, b, T(np.zeros(g.nc)), opts=o)
    assert rc == 0
    assert rel(lam.cpu().numpy(), z["lam_cert"]) <= TOL_LAM
    assert rep.hi_mvps == rep.iterations + 1 + rep.iterations // 20


# ------------------------------------------------------------------ GMRES recycling (NEXT-3)
def test_gmres_recycling_same_result_fewer_iterations(bp):
    """Recycled initial guesses change the iteration count, not the MVP (to tolerance):
    w(l3) for l3 = l1 + 0.5 l2 after solving l1 and l2 equals the cold solve, and a
    repeated right-hand side converges in at most a couple of Arnoldi iterations."""
    z = fixture(2)
    from synth import lambda_test
    g = bp.Geometry(z["centers"], int(z["p"]))
    bp.contacts(g, 0.1)
    l1, l2 = lambda_test(2, g.nc, 0), lambda_test(2, g.nc, 1)
    l3 = l1 + 0.5 * l2
    cold = bp.default_gmres_opts(tol=1e-12)
    w3, st_cold = bp.lcp_mvp(g, T(l3), gmres=cold)
    warm = bp.default_gmres_opts(tol=1e-12, recycle=1)
    bp.gmres_recycle_reset(g)
    bp.lcp_mvp(g, T(l1), gmres=warm)
    bp.lcp_mvp(g, T(l2), gmres=warm)
    w3r, st_warm = bp.lcp_mvp(g, T(l3), gmres=warm)
    assert rel(w3r.cpu().numpy(), w3.cpu().numpy()) <= TOL_VEL
    assert st_warm.iters < st_cold.iters
    w1r, st1 = bp.lcp_mvp(g, T(l1), gmres=warm)
    assert st1.iters <= 2 and rel(w1r.cpu().numpy(), z["w_test"][0]) <= TOL_VEL
    bp.gmres_recycle_reset(g)
    _, st_reset = bp.lcp_mvp(g, T(l3), gmres=warm)
    assert abs(st_reset.iters - st_cold.iters) <= 1   # fp64 atomics: summation order may differ


def test_gmres_recycling_spans_rhs_space(bp):
    """An LCP's MVP right-hand sides are linear in lambda (<= Nc dimensions): once the store
    holds Nc independent solves (c1: Nc = 12), any further MVP starts from an exact guess,
    converges in a few iterations (the stored solves' own 1e-12 residuals combine) instead of
    ~60 cold, and equals the oracle's A lambda (the store's capacity, up to 1024 pairs,
    exceeds Nc)."""
    z = fixture(1)
    g = bp.Geometry(z["centers"], int(z["p"]))
    bp.contacts(g, 0.1)
    warm = bp.default_gmres_opts(tol=1e-12, recycle=1)
    bp.gmres_recycle_reset(g)
    rng = np.random.default_rng(3)
    for _ in range(g.nc):
        bp.lcp_mvp(g, T(rng.uniform(0.0, 1.0, g.nc)), gmres=warm)
    lam = rng.uniform(0.0, 1.0, g.nc)
    w, st = bp.lcp_mvp(g, T(lam), gmres=warm)
    _, st_cold = bp.lcp_mvp(g, T(lam), gmres=bp.default_gmres_opts(tol=1e-12))
    assert st.iters <= 6 and st.iters * 5 < st_cold.iters, (st.iters, st_cold.iters)
    assert rel(w.cpu().numpy(), z["A_dense"] @ lam) <= TOL_VEL


@pytest.mark.parametrize("c", [1, 2])
def test_solve_lcp_bb_pgd(bp, c):
    """BB-PGD (method 2) on the device MVP reaches the unique LCP solution (R30)."""
    z = fixture(c)
    ref = z["lam_brute"] if c == 1 else z["lam_mono"]
    g = bp.Geometry(z["centers"], int(z["p"]))
    bp.contacts(g, 0.1)
    o = bp.default_solve_opts(method=2, eps_kkt_abs=1e-10, k_max=2000)
    o.gm_hi.tol = 1e-12
    lam, rep, rc = bp.solve_lcp(g, None, T(z["b"]), T(np.zeros(g.nc)), opts=o)
    assert rc == 0
    assert rel(lam.cpu().numpy(), ref) <= TOL_LAM
    assert rep.kkt_abs <= TOL_KKT
    assert rep.hi_mvps == rep.iterations + 1


# ------------------------------------------------------------------ DVI time step (NEXT-2)
def test_dvi_steps_vs_oracle(bp):
    """Two forward-Euler DVI steps through bpqn_dvi_step -- contacts, Janus-slip
    mobility, LCP, M D lambda, Euler update and bpqn_geometry_update -- against oracle/dvi.py."""
    from oracle import dvi
    C0 = np.array([[0.0, 0.0, 0.0], [2.03, 0.05, 0.0], [4.07, -0.05, 0.04]])
    ax0 = np.array([[0.0, 0.6, 0.8], [1.0, 0.0, 0.0], [0.0, -0.8, 0.6]])
    F = np.array([[3.0, 0.0, 0.0], [0.0, 0.0, 0.0], [-3.0, 0.0, 0.0]])
    p, dt = 6, 0.2
    hi = bp.Geometry(C0, p)
    o = bp.default_solve_opts(method=0, eps_kkt_abs=1e-12)
    o.gm_hi.tol = 1e-12
    C, ax = C0.copy(), ax0.copy()
    Co, axo = C0.copy(), ax0.copy()
    active = 0
    for step in range(2):
        uo, rep, rc = bp.dvi_step(hi, None, C, ax, F, slip_B=1.0, dt=dt, delta=0.1, opts=o)
        assert rc == 0
        Cn, an, Uo, lam, pairs = dvi.dvi_step(Co, axo, F, p=p, dt=dt, slip_B=1.0)
        assert rep.n_contacts == len(pairs)
        assert rep.active_contacts == int((lam > 0).sum())
        assert rel(uo, Uo) <= 1e-7
        assert rel(C - Co, Cn - Co) <= 1e-7
        np.testing.assert_allclose(ax, an, atol=1e-9)
        Co, axo = Cn, an
        active += rep.active_contacts
    assert active > 0                      # the LCP branch is exercised (step 2 has a live contact)
    assert rep.min_gap_after > 0


def test_gmres_not_converged_reported(bp):
    """max_iters reached before the tolerance -> BPQN_ERR_NOCONV (4), with the iterate and the
    achieved residual still returned through the stats (bpqn.h conventions)."""
    z = fixture(1)
    g = bp.Geometry(z["centers"], int(z["p"]))
    bp.contacts(g, 0.1)
    from synth import lambda_test
    with pytest.raises(bp.BpqnError) as e:
        bp.lcp_mvp(g, T(lambda_test(1, g.nc, 0)), gmres=bp.default_gmres_opts(tol=1e-14, max_iters=5))
    assert e.value.code == 4
    _, st = bp.mobility_apply(g, T(z["FT_test"]), gmres=bp.default_gmres_opts(tol=1e-6))
    assert 1 <= st.iters < 60 and st.rel_resid <= 1e-6 and st.applies >= st.iters


def test_bi_pqn_inexact_subproblems_same_solution(bp):
    """The sub_forcing option changes the work, not the LCP solution (unique, R30)."""
    z = fixture(2)
    g = bp.Geometry(z["centers"], int(z["p"]))
    pr, nr, gp = bp.contacts(g, 0.1)
    lo = bp.Geometry(z["centers"], int(z["p_lo"]))
    bp.set_contacts(lo, pr, nr, gp)
    o = bp.default_solve_opts(method=1, eps_kkt_abs=1e-10, sub_forcing=0.1)
    o.gm_hi.tol = 1e-12
    o.gm_lo.tol = 1e-12
    lam, rep, rc = bp.solve_lcp(g, lo, T(z["b"]), T(np.zeros(g.nc)), opts=o)
    assert rc == 0
    assert rel(lam.cpu().numpy(), z["lam_bi"]) <= TOL_LAM
    assert rep.lo_mvps <= int(z["bi_lo_mvps"])


def test_geometry_update_equals_fresh_init(bp):
    """bpqn_geometry_update (kept self operators, rebuilt near data) == a fresh handle."""
    from synth import layer_densities, make_config
    cfg = make_config(2)
    C1 = 1.01 * cfg["centers"] + np.array([0.3, -0.2, 0.1])   # dilate + shift: gaps grow, near sets change
    g = bp.Geometry(cfg["centers"], cfg["p"])
    bp.geometry_update(g, C1)
    h = bp.Geometry(C1, cfg["p"])
    f, q = layer_densities(2, g.N)
    u1 = bp.layer_apply(g, T(f), T(q)).cpu().numpy()
    u2 = bp.layer_apply(h, T(f), T(q)).cpu().numpy()
    assert rel(u1, u2) <= 1e-13
    with pytest.raises(bp.BpqnError) as e:          # overlapping update is rejected
        C2 = C1.copy()
        C2[1] = C2[0] + np.array([1.9, 0.0, 0.0])
        bp.geometry_update(g, C2)
    assert e.value.code == 1


def test_dvi_step_bi_pqn_vs_oracle(bp):
    """One DVI step with the Bi-PQN solver (hi p = 6, lo p = 4 handles moved together)."""
    from oracle import dvi
    C0 = np.array([[0.0, 0.0, 0.0], [2.03, 0.05, 0.0], [4.07, -0.05, 0.04]])
    ax0 = np.array([[0.0, 0.6, 0.8], [1.0, 0.0, 0.0], [0.0, -0.8, 0.6]])
    F = np.array([[12.0, 0.0, 0.0], [0.0, 0.0, 0.0], [-12.0, 0.0, 0.0]])
    hi, lo = bp.Geometry(C0, 6), bp.Geometry(C0, 4)
    o = bp.default_solve_opts(method=1, eps_kkt_abs=1e-12)
    o.gm_hi.tol = o.gm_lo.tol = 1e-12
    C, ax = C0.copy(), ax0.copy()
    uo, rep, rc = bp.dvi_step(hi, lo, C, ax, F, slip_B=1.0, dt=0.2, delta=0.1, opts=o)
    assert rc == 0 and rep.active_contacts > 0 and rep.lcp.lo_mvps > 0
    Cn, an, Uo, lam, pairs = dvi.dvi_step(C0, ax0, F, p=6, dt=0.2, slip_B=1.0)
    assert rel(C - C0, Cn - C0) <= 1e-7
    np.testing.assert_allclose(ax, an, atol=1e-9)
    # both handles now sit at the new centres: a fresh hi handle gives the same operator
    f = np.random.default_rng(2).standard_normal((hi.N, 3))
    fresh = bp.Geometry(C, 6)
    assert rel(bp.layer_apply(hi, T(f)).cpu().numpy(), bp.layer_apply(fresh, T(f)).cpu().numpy()) <= 1e-13


def test_plain_c_client(bp):
    """examples/bpqn_mvp (pure C against include/bpqn.h) gives the binding's MVP."""
    import json
    import subprocess
    exe = os.path.join(ROOT, "examples", "bpqn_mvp")
    if not os.path.exists(exe):
        from paper_2604_10089_b200 import build as b
        b.build_example()
    out = json.loads(subprocess.check_output([exe, "6"], timeout=300).decode().strip().splitlines()[-1])
    C = np.array([[2.05 * i + 0.01 * l, 2.05 * j - 0.01 * i, 2.05 * l + 0.005 * j]
                  for i in range(2) for j in range(2) for l in range(2)])
    g = bp.Geometry(C, 6)
    bp.contacts(g, 0.1)
    assert g.nc == out["n_contacts"]
    w, st = bp.lcp_mvp(g, T(1.0 / (1 + np.arange(g.nc))))
    assert abs(np.linalg.norm(w.cpu().numpy()) - out["w_norm"]) <= 1e-9 * out["w_norm"]
    assert out["hi_mvps"] == out["lcp_iterations"] + 1 + out["lcp_iterations"] // 20
    assert out["kkt_abs"] <= 1e-10


# ------------------------------------------------------------------ full-size properties (c4)
def _rot_z(t):
    c, s = np.cos(t), np.sin(t)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


@pytest.mark.parametrize("kind", ["translation", "rotation_pi_over_p"])
def test_lcp_mvp_c4_exact_covariance(bp, kind):
    """At full c4 size, in the bench's launch configuration: the discrete operator is exactly
    covariant under translations and under the rotation by pi/p about z, which maps every
    sphere's grid onto itself -- so w = D^T M D lambda (a scalar per contact) is
    unchanged to GMRES tolerance.  No oracle needed: a property at any size."""
    from synth import lambda_test, make_config
    cfg = make_config(4)
    C = cfg["centers"]
    if kind == "translation":
        C2 = C + np.array([3.7, -1.1, 0.4])
    else:
        C2 = C @ _rot_z(np.pi / cfg["p"]).T
    gm = bp.default_gmres_opts(tol=1e-12)
    ws = []
    for cc in (C, C2):
        g = bp.Geometry(cc, cfg["p"])
        bp.contacts(g, 0.1)
        w, st = bp.lcp_mvp(g, T(lambda_test(4, g.nc, 0)), gmres=gm)
        ws.append(w.cpu().numpy())
        del g
    assert rel(ws[1], ws[0]) <= 1e-10


def test_shard_argument_errors(bp):
    """bpqn_geometry_shard / _symmetric reject bad ranks and an unsharded handle (code 1)."""
    import ctypes
    C, p = _scene("two_near_p6")
    g = bp.Geometry(C, p)
    L = bp.lib()
    cb = bp._bpqn.ALLGATHER_FN(lambda _u: 0)
    buf = ctypes.c_void_p(1)
    assert L.bpqn_geometry_shard(g.h, 2, 2, buf, buf, cb, None) == 1          # rank >= world
    assert L.bpqn_geometry_shard(g.h, 0, 3, buf, buf, cb, None) == 1          # more ranks than spheres
    assert L.bpqn_geometry_shard_symmetric(g.h, buf, buf, cb, None) == 1      # not sharded
    assert L.bpqn_geometry_shard_symmetric(g.h, None, None, bp._bpqn.ALLGATHER_FN(0), None) == 0  # disable: ok


# ------------------------------------------------------------------ determinism and the GMRES cycle graph
def _cfg_geometry(bp, c):
    from synth import make_config
    cfg = make_config(c)
    g = bp.Geometry(cfg["centers"], cfg["p"])
    bp.contacts(g, cfg["delta"])
    return g, cfg


@pytest.mark.parametrize("c", [1, 2])
def test_operator_and_mvp_bit_reproducible(bp, c):
    """No floating-point atomics on the path (fixed-order K1/K2/K3 partial sums, K1-K4):
    the layer operator and the LCP MVP give bit-identical results run to run.  The first MVP on a
    handle runs its GMRES steps host-driven, later ones replay the captured cycle graph (conditional
    WHILE node): identical bits mean the graph runs exactly the same kernels."""
    import torch
    from synth import lambda_test
    g, cfg = _cfg_geometry(bp, c)
    rng = np.random.default_rng(7)
    f, q = T(rng.standard_normal((g.N, 3))), T(rng.standard_normal((g.N, 3)))
    u1 = bp.layer_apply(g, f, q).cpu().numpy()
    u2 = bp.layer_apply(g, f, q).cpu().numpy()
    assert np.array_equal(u1, u2)
    lam = T(lambda_test(c, g.nc, 0))
    gm = bp.default_gmres_opts(tol=1e-10)
    ws, its = [], []
    for _ in range(3):
        w, st = bp.lcp_mvp(g, lam, gmres=gm)
        torch.cuda.synchronize()
        ws.append(w.cpu().numpy())
        its.append(st.iters)
    assert len(set(its)) == 1, its
    assert np.array_equal(ws[0], ws[1]) and np.array_equal(ws[1], ws[2])


def test_gmres_restart_cycles_match_unrestarted(bp):
    """Restarted GMRES(m) with the device-side stopping test: a short restart length (several
    cycles, each its own graph launch) reaches the same solution as one long cycle."""
    from synth import lambda_test
    g, cfg = _cfg_geometry(bp, 1)
    lam = T(lambda_test(1, g.nc, 1))
    w_long, st_long = bp.lcp_mvp(g, lam, gmres=bp.default_gmres_opts(tol=1e-12, restart=200))
    w_short, st_short = bp.lcp_mvp(g, lam, gmres=bp.default_gmres_opts(tol=1e-12, restart=7))
    w_short2, st_short2 = bp.lcp_mvp(g, lam, gmres=bp.default_gmres_opts(tol=1e-12, restart=7))
    assert st_short.restarts >= 2 and st_long.restarts == 0
    assert rel(w_short.cpu().numpy(), w_long.cpu().numpy()) < 1e-10
    assert np.array_equal(w_short.cpu().numpy(), w_short2.cpu().numpy())
    assert st_short.iters == st_short2.iters


def test_rsqrt_seed_bound_exhaustive(bp):
    """K1 and K2 take rho^-k from the MUFU.RSQ64H seed y and the series (1 - e)^(-k/2) truncated
    after e^2 (allpairs.cu); the truncation error (< 7 |e|^3 relative for k <= 5) is
    negligible only if |e| = |1 - rho^2 y^2| <= 2^-19.  Exhaustive over every high-word input pattern
    of rho^2 = 2^e (1 + m) for e in [-60, 210] (near-contact pairs at gap 1e-4 up to the 1e30 padding
    records), both low-word extremes: the bound holds (measured max |e| = 1.8596e-6 < 2^-19 = 1.907e-6),
    so the truncated series is accurate to 7 |e|^3 < 4.6e-17 relative."""
    from paper_2604_10089_b200 import _bpqn
    e = _bpqn.diag_rsqrt_seed(-60, 210)
    assert 0 < e <= 2.0 ** -19, e
    assert 7 * e ** 3 < 4.6e-17


def test_solve_lcp_dense_dev_c1(bp):
    """bpqn_solve_lcp_dense_dev (device arrays + stream) on the oracle's densified c1
    LCP matrix: Mono-PQN and Bi-PQN (A^ = A perturbed) reach the brute-force solution (O14)."""
    import torch
    z = fixture(1)
    A, b = T(z["A_dense"]), T(z["b"])
    for method, Ahat in ((0, None), (1, T(z["A_dense"] * 1.05))):
        x = torch.zeros(b.shape[0], dtype=torch.float64, device="cuda")
        x, rep, rc = bp._bpqn.solve_lcp_dense_dev(A, b, x, Ahat=Ahat,
                                                  opts=bp.default_solve_opts(method=method, eps_kkt_abs=1e-12))
        assert rc == 0
        assert rel(x.cpu().numpy(), z["lam_brute"]) <= TOL_LAM


# ------------------------------------------------------------------ dense LCP matrix / densified low fidelity (R38)
@pytest.mark.parametrize("c,p", [(1, 8), (2, 6)])
def test_lcp_matrix_dense_equals_mvps(bp, c, p):
    """bpqn_lcp_matrix_dense (all Nc mobility solves as one batched GMRES on the assembled dense
    operator, cuBLAS DGEMM) equals the matrix-free LCP MVP on every unit vector (c1 at p = 8, the c2
    low fidelity p = 6) to the GMRES tolerance, and at c1 the oracle's densified A."""
    import torch
    from synth import make_config
    cfg = make_config(c)
    g = bp.Geometry(cfg["centers"], p)
    bp.contacts(g, cfg["delta"])
    gm = bp.default_gmres_opts(tol=1e-12)
    A, st = bp.lcp_matrix_dense(g, gmres=gm)
    cols = []
    for l in range(g.nc):
        e = torch.zeros(g.nc, dtype=torch.float64, device="cuda")
        e[l] = 1.0
        w, _ = bp.lcp_mvp(g, e, gmres=gm)
        cols.append(w.cpu().numpy())
    Amf = np.stack(cols, axis=1)
    assert rel(A, Amf) <= 1e-10, rel(A, Amf)
    if c == 1:
        assert rel(A, fixture(1)["A_dense"]) <= TOL_VEL


@pytest.mark.parametrize("c,p", [(1, 8), (2, 6)])
def test_lcp_matrix_dense_block_equals_batched(bp, c, p):
    """The block GMRES that forms A^ by default (one Krylov space for all Nc columns, normal equations of
    the block Hessenberg with one refinement step) equals the batched per-column GMRES
    (BPQN_LO_BATCHED=1) to the GMRES tolerance, in fewer operator applications."""
    from synth import make_config
    cfg = make_config(c)
    g = bp.Geometry(cfg["centers"], p)
    bp.contacts(g, cfg["delta"])
    for tol in (1e-6, 1e-12):
        gm = bp.default_gmres_opts(tol=tol)
        Ab, stb = bp.lcp_matrix_dense(g, gmres=gm)
        os.environ["BPQN_LO_BATCHED"] = "1"
        try:
            Aa, sta = bp.lcp_matrix_dense(g, gmres=gm)
        finally:
            del os.environ["BPQN_LO_BATCHED"]
        assert rel(Ab, Aa) <= 100 * tol, (tol, rel(Ab, Aa))
        assert stb.iters < sta.iters, (stb.iters, sta.iters)
    # restarted block GMRES (3 block iterations per cycle, restarts from the true residual)
    os.environ["BPQN_LO_BLOCK_KMAX"] = "3"
    try:
        Ar, str_ = bp.lcp_matrix_dense(g, gmres=bp.default_gmres_opts(tol=1e-10))
    finally:
        del os.environ["BPQN_LO_BLOCK_KMAX"]
    assert str_.iters > 3 and rel(Ar, Aa) <= 1e-8, (str_.iters, rel(Ar, Aa))


def test_solve_lcp_bi_dense_lo_c2(bp):
    """Bi-PQN with the low-fidelity LCP matrix formed once (lo_dense = 1, R38) reaches the oracle's
    lambda* at c2 (<= 1e-7) with the oracle-A complementarity (R26) <= 1e-8; every low-fidelity MVP
    is then an Nc x Nc product."""
    z = fixture(2)
    g = bp.Geometry(z["centers"], int(z["p"]))
    pr, nr, gp = bp.contacts(g, 0.1)
    lo = bp.Geometry(z["centers"], int(z["p_lo"]))
    bp.set_contacts(lo, pr, nr, gp)
    o = bp.default_solve_opts(method=1, eps_kkt_abs=1e-10, lo_dense=1)
    o.gm_hi.tol = 1e-12
    o.gm_lo.tol = 1e-12
    lam, rep, rc = bp.solve_lcp(g, lo, T(z["b"]), T(np.zeros(g.nc)), opts=o)
    assert rc == 0
    assert rep.lo_dense_columns == g.nc and rep.lo_mvps > 0
    assert rel(lam.cpu().numpy(), z["lam_bi"]) <= TOL_LAM
    if "A_dense" in z:
        assert _kkt(lam.cpu().numpy(), z["A_dense"], z["b"]) <= TOL_KKT


@pytest.mark.parametrize("cfg", [0, 3, 4, 6, 11, 14, 15, 16, 19, 22])
def test_k1_launch_shapes_agree(bp, cfg):
    """Every selectable symmetric-K1 launch shape (BPQN_K1_CFG) equals the one-directional
    kernel (BPQN_K1=asym) on c1 and c2 for S, D and S+D layer applies (a 4-warp shape once dropped the
    source-side sums of the tile rows its 128 threads did not cover)."""
    import subprocess
    import sys
    tool = os.path.join(ROOT, "tools", "k1_cfg_check.py")
    for c in (1, 2):
        out = subprocess.run([sys.executable, tool, "--config", str(c), "--cfgs", str(cfg)], capture_output=True,
                             text=True, timeout=600)
        assert out.returncode == 0, out.stderr[-2000:]
        line = [l for l in out.stdout.splitlines() if l.startswith("cfg")][-1]
        errs = [float(x) for x in line.split("{")[1].replace("'", "").replace("}", "").replace(",", "").split()
                if x[0].isdigit()]
        assert len(errs) == 3 and max(errs) <= 1e-12, line


@pytest.mark.parametrize("p,gap,axis", [(2, 0.05, "x"), (5, 1e-3, "z"), (8, 0.01, "rand"), (16, 0.02, "z"),
                                        (16, 0.3, "rand"), (24, 0.004, "rand")])
def test_near_rotation_equals_brute_force(bp, p, gap, axis):
    """The rotation form of the near rule (k_near_rot: axisymmetric theta' integrals x second-order
    jets of the rotated SH basis) equals the point-by-point refined rule (k_quad_rows, selected by
    BPQN_NEAR_BRUTE=1) -- the same discrete operator, so S, D and S+D applies agree to rounding.
    Targets next to the grid poles (axis z) exercise the frame construction."""
    rng = np.random.default_rng(p)
    e = {"x": np.array([1.0, 0, 0]), "z": np.array([0, 0, 1.0])}.get(axis)
    if e is None:
        e = rng.standard_normal(3)
        e /= np.linalg.norm(e)
    C = np.array([[0.1, -0.2, 0.3], [0.1, -0.2, 0.3] + (2.0 + gap) * e, [0.1, -0.2, 0.3] - (2.0 + 3 * gap) * e])
    os.environ["BPQN_NEAR_BRUTE"] = "1"
    try:
        gb = bp.Geometry(C, p)
    finally:
        del os.environ["BPQN_NEAR_BRUTE"]
    gr = bp.Geometry(C, p)
    assert gr.n_incidences == gb.n_incidences > 0
    f, q = rng.standard_normal((gr.N, 3)), rng.standard_normal((gr.N, 3))
    for kw in (dict(f=T(f)), dict(q=T(q)), dict(f=T(f), q=T(q))):
        ur = bp.layer_apply(gr, **kw).cpu().numpy()
        ub = bp.layer_apply(gb, **kw).cpu().numpy()
        assert rel(ur, ub) <= 1e-13, (list(kw), rel(ur, ub))


# ------------------------------------------------------------------ NEXT-4: FMM far field (fmm_order)
def torch_equal(a, b):
    import torch
    return bool(torch.equal(a, b))


def _lattice(n, seed, spacing=2.02, jitter=0.01):
    rng = np.random.default_rng(seed)
    g1 = np.arange(n) * spacing
    return np.array([[x, y, z] for x in g1 for y in g1 for z in g1]) + rng.uniform(-jitter, jitter, (n ** 3, 3))


def _fmm_geometry(bp, C, p, order, levels=None):
    op = bp.default_disc_opts()
    op.fmm_order = order
    if levels:
        os.environ["BPQN_FMM_LEVELS"] = str(levels)
    try:
        return bp.Geometry(C, p, opts=op)
    finally:
        os.environ.pop("BPQN_FMM_LEVELS", None)


@pytest.mark.parametrize("levels", [2, 3, 4])
def test_fmm_layer_apply_vs_direct(bp, levels):
    """The FMM far field (order 10) against the direct all-pairs K1 on the same geometry: S, D and S+D layer
    applies within the measured FMM accuracy (order 10: ~3e-8 S, ~2e-7 D; bound 1e-6), with 2, 3 and 4 tree
    levels (M2M / L2L exercised); two applies are bit-identical."""
    C = _lattice(6, 41)
    gd = bp.Geometry(C, 6)
    gf = _fmm_geometry(bp, C, 6, 10, levels)
    rng = np.random.default_rng(42)
    f, q = T(rng.standard_normal((gd.N, 3))), T(rng.standard_normal((gd.N, 3)))
    for kw in (dict(f=f), dict(q=q), dict(f=f, q=q)):
        ud = bp.layer_apply(gd, **kw).cpu().numpy()
        uf = bp.layer_apply(gf, **kw).cpu().numpy()
        assert rel(uf, ud) <= 1e-6, (list(kw), rel(uf, ud))
    u1 = bp.layer_apply(gf, f=f, q=q).cpu().numpy()
    u2 = bp.layer_apply(gf, f=f, q=q).cpu().numpy()
    assert np.array_equal(u1, u2)


@pytest.mark.parametrize("order,levels,bound", [(6, 3, 6e-4), (6, 4, 6e-4), (8, 3, 2e-5), (5, 3, 6e-3)])
def test_fmm_low_orders_skeleton_m2l(bp, order, levels, bound):
    """Orders 5-8 apply M2L through shared row / column skeletons (tolerance about the order's own far-field
    error), small leaves run the equal-cost leaf items, M2M / L2L are grouped over the 8 octants (4 levels): S, D
    and S+D layer applies stay within the order's accuracy of the direct K1 sum, the compressed operator differs
    from the exact-M2L one (BPQN_FMM_M2L_TOL=0) by no more than that, and two applies are bit-identical."""
    C = _lattice(6, 51)
    gd = bp.Geometry(C, 8)
    gf = _fmm_geometry(bp, C, 8, order, levels)
    os.environ["BPQN_FMM_M2L_TOL"] = "0"
    try:
        gx = _fmm_geometry(bp, C, 8, order, levels)
    finally:
        os.environ.pop("BPQN_FMM_M2L_TOL", None)
    rng = np.random.default_rng(52)
    f, q = T(rng.standard_normal((gd.N, 3))), T(rng.standard_normal((gd.N, 3)))
    for kw in (dict(f=f), dict(q=q), dict(f=f, q=q)):
        ud = bp.layer_apply(gd, **kw).cpu().numpy()
        uf = bp.layer_apply(gf, **kw).cpu().numpy()
        ux = bp.layer_apply(gx, **kw).cpu().numpy()
        assert rel(ux, ud) <= bound, (list(kw), rel(ux, ud))
        assert rel(uf, ud) <= bound, (list(kw), rel(uf, ud))
        assert rel(uf, ux) <= bound, (list(kw), rel(uf, ux))
    u1 = bp.layer_apply(gf, f=f, q=q).cpu().numpy()
    u2 = bp.layer_apply(gf, f=f, q=q).cpu().numpy()
    assert np.array_equal(u1, u2)


@pytest.mark.parametrize("scene", ["c3_rsa", "single", "two_far"])
def test_fmm_sparse_trees(bp, scene):
    """FMM on trees with many empty boxes: the c3 random sequential packing (64 spheres, 3 levels), one sphere,
    two spheres far apart (most boxes empty, leaves with points only at two corners)."""
    from synth import make_config
    if scene == "c3_rsa":
        C, p, lv = make_config(3)["centers"], 6, 3
    elif scene == "single":
        C, p, lv = np.array([[0.3, -0.2, 0.1]]), 8, 2
    else:
        C, p, lv = np.array([[0.0, 0.0, 0.0], [9.0, 7.5, -6.0]]), 8, 3
    gd = bp.Geometry(C, p)
    gf = _fmm_geometry(bp, C, p, 10, lv)
    rng = np.random.default_rng(48)
    f, q = T(rng.standard_normal((gd.N, 3))), T(rng.standard_normal((gd.N, 3)))
    ud = bp.layer_apply(gd, f=f, q=q).cpu().numpy()
    uf = bp.layer_apply(gf, f=f, q=q).cpu().numpy()
    # one sphere: every far pair lies on the same sphere and the sum cancels more (|u| ~ 1/4 of the
    # multi-sphere scenes'), so the FMM's error relative to |u| is larger
    assert rel(uf, ud) <= (5e-6 if scene == "single" else 1e-6), rel(uf, ud)


def test_fmm_layer_apply_vs_oracle(bp):
    """FMM-mode layer apply (order 10, 3 levels) against the oracle's direct operator on sampled targets."""
    from oracle.layer import Disc
    C = _lattice(4, 43)
    d = Disc(C, 5)
    g = _fmm_geometry(bp, C, 5, 10, 3)
    rng = np.random.default_rng(44)
    f, q = rng.standard_normal((d.N, 3)), rng.standard_normal((d.N, 3))
    u = bp.layer_apply(g, f=T(f), q=T(q)).cpu().numpy()
    tg = _sample_targets(d, 48, 45)
    assert rel(u[tg], d.apply(f=f, q=q, targets=tg)) <= 1e-6


def test_fmm_lcp_mvp_vs_direct(bp):
    """An LCP MVP (GMRES 1e-10) with the FMM far field equals the direct one to the FMM accuracy."""
    C = _lattice(4, 46)
    gd = bp.Geometry(C, 6)
    gf = _fmm_geometry(bp, C, 6, 10, 2)
    bp.contacts(gd, 0.1)
    bp.contacts(gf, 0.1)
    assert gd.nc == gf.nc > 0
    lam = T(np.random.default_rng(47).uniform(0, 1, gd.nc))
    gm = bp.default_gmres_opts(tol=1e-10)
    wd, _ = bp.lcp_mvp(gd, lam, gmres=gm)
    wf, _ = bp.lcp_mvp(gf, lam, gmres=gm)
    assert rel(wf.cpu().numpy(), wd.cpu().numpy()) <= 1e-5
    # later MVPs replay the captured GMRES cycle graph (cuBLAS M2L GEMMs inside the capture): bit-identical
    for _ in range(2):
        w2, _ = bp.lcp_mvp(gf, lam, gmres=gm)
        assert torch_equal(w2, wf)


def test_fmm_geometry_update_equals_fresh(bp):
    """bpqn_geometry_update on an FMM handle rebuilds the tree and lists: it equals a fresh FMM handle at the
    new centres bit for bit (the unit-box operators are kept)."""
    C = _lattice(4, 49)
    C1 = 1.01 * C + np.array([0.2, -0.1, 0.3])
    g = _fmm_geometry(bp, C, 6, 8)
    bp.geometry_update(g, C1)
    h = _fmm_geometry(bp, C1, 6, 8)
    rng = np.random.default_rng(50)
    f, q = T(rng.standard_normal((g.N, 3))), T(rng.standard_normal((g.N, 3)))
    assert np.array_equal(bp.layer_apply(g, f=f, q=q).cpu().numpy(), bp.layer_apply(h, f=f, q=q).cpu().numpy())


def test_fmm_bi_pqn_solve_matches_direct(bp):
    """A Bi-PQN LCP solve whose high fidelity uses the FMM far field (order 10) reaches the direct solve's
    lambda* to the FMM accuracy (the LCP is strongly monotone: a perturbed A moves lambda* by
    O(|dA|), Lemma 2)."""
    C = _lattice(4, 51, spacing=2.03, jitter=0.015)
    gd = bp.Geometry(C, 6)
    gf = _fmm_geometry(bp, C, 6, 10, 2)
    lo = bp.Geometry(C, 4)
    pr, nr, gp = bp.contacts(gd, 0.1)
    bp.set_contacts(gf, pr, nr, gp)
    bp.set_contacts(lo, pr, nr, gp)
    b = T(np.random.default_rng(52).uniform(-0.05, 0.02, gd.nc))
    out = []
    for g in (gd, gf):
        o = bp.default_solve_opts(method=1, eps_kkt_abs=1e-10)
        o.gm_hi.tol = 1e-11
        o.gm_lo.tol = 1e-11
        lam, rep, rc = bp.solve_lcp(g, lo, b, T(np.zeros(gd.nc)), opts=o)
        assert rc == 0
        out.append(lam.cpu().numpy())
    assert rel(out[1], out[0]) <= 1e-5, rel(out[1], out[0])


# ------------------------------------------------------------------ FMM-accelerated refinement (relax_fmm)
@pytest.mark.parametrize("c", [1, 2])
def test_fmm_refinement_mvp_vs_oracle(bp, c):
    """FMM refinement (bpqn_gmres_opts.relax_fmm, order 6 -- the least accurate order used): every Krylov step
    with the FMM far field, every cycle from the direct residual.  The LCP MVP meets the PARITY bar against the
    oracle fixture at the parity tolerance 1e-12 (the returned x meets tol for the direct operator), several
    refinement cycles ran, and only the residuals used the direct operator."""
    z = fixture(c)
    C, p = z["centers"], int(z["p"])
    g = _fmm_geometry(bp, C, p, 6, 2)
    bp.contacts(g, 0.1)
    from synth import lambda_test
    lam = lambda_test(c, g.nc, 0)
    w, st = bp.lcp_mvp(g, T(lam), gmres=bp.default_gmres_opts(tol=1e-12, relax_fmm=1))
    assert st.fmm_applies == st.iters and st.applies == st.iters + st.restarts, (st.iters, st.applies)
    assert st.restarts >= 2 and st.rel_resid <= 1e-12
    assert rel(w.cpu().numpy(), z["w_test"][0]) <= TOL_VEL, (st.iters, st.restarts)


def test_fmm_refinement_matches_direct_gmres(bp):
    """FMM refinement vs plain GMRES on a direct handle at tol 1e-10 and several cycle reductions delta: the MVPs
    agree to the tolerance level; the captured cycle graph replays bit-identically; without relax_fmm an FMM
    handle uses the FMM throughout; relax_fmm on a direct handle is an argument error."""
    C = _lattice(4, 61)
    gd = bp.Geometry(C, 6)
    gf = _fmm_geometry(bp, C, 6, 6, 2)
    bp.contacts(gd, 0.1)
    bp.contacts(gf, 0.1)
    lam = T(np.random.default_rng(62).uniform(0, 1, gd.nc))
    wd, sd = bp.lcp_mvp(gd, lam, gmres=bp.default_gmres_opts(tol=1e-10))
    for delta in (0.0, 1e-2, 1e-4):
        wr, sr = bp.lcp_mvp(gf, lam, gmres=bp.default_gmres_opts(tol=1e-10, relax_fmm=1, relax_delta=delta))
        assert sr.fmm_applies == sr.iters > 0 and sr.restarts >= 1 and sr.rel_resid <= 1e-10, delta
        assert rel(wr.cpu().numpy(), wd.cpu().numpy()) <= 1e-8, delta
    gm = bp.default_gmres_opts(tol=1e-10, relax_fmm=1)
    w1, _ = bp.lcp_mvp(gf, lam, gmres=gm)
    w2, _ = bp.lcp_mvp(gf, lam, gmres=gm)
    assert torch_equal(w1, w2)
    _, s0 = bp.lcp_mvp(gf, lam, gmres=bp.default_gmres_opts(tol=1e-10))
    assert s0.fmm_applies == s0.applies
    with pytest.raises(bp.BpqnError):
        bp.lcp_mvp(gd, lam, gmres=bp.default_gmres_opts(tol=1e-10, relax_fmm=1))


def test_fmm_refinement_bi_pqn_solve_matches_direct(bp):
    """A Bi-PQN LCP solve whose high-fidelity MVPs use FMM refinement reaches the direct solve's lambda* to the
    solve tolerance (each MVP meets the GMRES tolerance for the direct operator)."""
    C = _lattice(4, 63, spacing=2.03, jitter=0.015)
    gd = bp.Geometry(C, 6)
    gf = _fmm_geometry(bp, C, 6, 6, 2)
    lo = bp.Geometry(C, 4)
    pr, nr, gp = bp.contacts(gd, 0.1)
    bp.set_contacts(gf, pr, nr, gp)
    bp.set_contacts(lo, pr, nr, gp)
    b = T(np.random.default_rng(64).uniform(-0.05, 0.02, gd.nc))
    out = []
    for g, rf in ((gd, 0), (gf, 1)):
        o = bp.default_solve_opts(method=1, eps_kkt_abs=1e-10)
        o.gm_hi.tol = 1e-11
        o.gm_hi.relax_fmm = rf
        o.gm_lo.tol = 1e-11
        lam, rep, rc = bp.solve_lcp(g, lo, b, T(np.zeros(gd.nc)), opts=o)
        assert rc == 0
        out.append(lam.cpu().numpy())
    assert np.max(np.abs(out[1] - out[0])) <= 1e-7 * max(1.0, np.max(np.abs(out[0])))
