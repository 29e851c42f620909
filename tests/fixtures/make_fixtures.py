"""Writes tests/fixtures/c{1..4}.npz -- every stored value comes from oracle/ only.

Usage: python tests/fixtures/make_fixtures.py [c ...] [--no-lcp]
       python tests/fixtures/make_fixtures.py --dense 2 3
--dense adds to an existing c2/c3 fixture the oracle's densified LCP matrices
(A = D^T M D column by column: one oracle MVP per unit vector, GMRES 1e-13; the
low-fidelity A^ likewise) and re-runs the oracle's Mono-/Bi-PQN on them (O14's
dense route; the matrix-free and dense operators agree to the GMRES tolerance).
The -m gpu tests then evaluate R26's complementarity residual with the oracle's A.
       python tests/fixtures/make_fixtures.py --certify 4 LAMBDA.npy
--certify stores a KKT certificate for a candidate solution lambda of the c4 LCP
(where the oracle cannot afford its own solve: Nc = 540 columns at ~1 h per oracle
MVP): the oracle's A lambda (one oracle MVP, GMRES 1e-13) and
||min(lambda, A lambda + b)||_2 with the oracle's A and b (R26).  lambda is only an
input to the oracle here; the stored expected values are the oracle's (R35).
The oracle's operator data are built first; the script then waits for LAMBDA.npy.
Runs the plain CPU oracle (oracle/) on the seeded synth/ inputs and stores the
operator outputs and LCP solutions the -m gpu parity tests compare against
(SURVEY 8(c).4).  Wall time and core count of each piece are recorded.
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import lcp, mobility as mob, native, pqn  # noqa: E402
from oracle.layer import Disc  # noqa: E402
from synth import ft_test, lambda_test, make_config  # noqa: E402

GMRES_TOL = 1e-13
EPS_KKT = 1e-10
N_LAMBDA = {1: 3, 2: 3, 3: 2, 4: 1}


def log(*a):
    print(time.strftime("%H:%M:%S"), *a, flush=True)


def run(c, do_lcp=True):
    cfg = make_config(c)
    out = dict(centers=cfg["centers"], axes=cfg["axes"], F_nc=cfg["F_nc"], p=cfg["p"],
               gmres_tol=GMRES_TOL, eps_kkt=EPS_KKT, cores=os.cpu_count())
    t0 = time.time()
    d = Disc(cfg["centers"], cfg["p"], cfg["radius"], cfg["mu"])
    pairs, nrm, gaps = lcp.contacts(cfg["centers"], cfg["radius"], cfg["delta"])
    out.update(pairs=pairs, normals=nrm, gaps=gaps, n_near_pairs=len(d.near), n_incidences=len(d.inc),
               inc_t=d.inc_t, inc_m=d.inc_m, ps=d.ps, dnear=d.dnear)
    log("c%d Np=%d N=%d Nc=%d near=%d inc=%d" % (c, d.np, d.N, len(pairs), len(d.near), len(d.inc)))
    times = {}
    t = time.time()
    FT = ft_test(c, d.np)
    UO, info = mob.mobility(d, FT, tol=GMRES_TOL, return_info=True)
    times["mobility"] = time.time() - t
    out.update(FT_test=FT, UO_test=UO, gmres_iters_mob=info["iters"])
    log("c%d mobility %.1fs iters %d" % (c, times["mobility"], info["iters"]))
    ws = []
    for k in range(N_LAMBDA[c]):
        t = time.time()
        lam = lambda_test(c, len(pairs), k)
        w, info = lcp.lcp_mvp(d, pairs, nrm, lam, tol=GMRES_TOL, return_info=True)
        times["mvp%d" % k] = time.time() - t
        ws.append(w)
        log("c%d mvp%d %.1fs iters %d" % (c, k, times["mvp%d" % k], info["iters"]))
    out["w_test"] = np.array(ws)
    t = time.time()
    slip = mob.janus_slip(d, cfg["axes"], cfg["slip_B"])
    b, U_nc = lcp.lcp_b(d, pairs, nrm, gaps, cfg["F_nc"], slip, tol=GMRES_TOL)
    times["b"] = time.time() - t
    out.update(b=b, U_nc=U_nc)
    log("c%d b %.1fs, negative fraction %.2f" % (c, times["b"], (b < 0).mean()))
    if do_lcp:
        A_hi = lambda v: lcp.lcp_mvp(d, pairs, nrm, v, tol=GMRES_TOL)
        if c == 1:
            t = time.time()
            A = lcp.densify(A_hi, len(pairs))
            lam_bf, cnt = lcp.brute_force_lcp(A, b)
            times["dense_bf"] = time.time() - t
            out.update(A_dense=A, lam_brute=lam_bf, brute_count=cnt)
            log("c1 brute force: %d accepted sets" % cnt)
        if cfg["solve"] in ("mono", "both"):
            t = time.time()
            x, g, _, _, rep = pqn.mono_pqn(lambda v: (A_hi(v), None), b, np.zeros(len(pairs)),
                                           eps_abs=EPS_KKT)
            times["mono"] = time.time() - t
            out.update(lam_mono=x, mono_iters=rep["iterations"], mono_mvps=rep["mvps"],
                       mono_kkt=rep["kkt_abs"], mono_term=rep["termination"])
            log("c%d mono-PQN iters %d mvps %d kkt %.2e %.1fs" % (c, rep["iterations"], rep["mvps"],
                                                                 rep["kkt_abs"], times["mono"]))
        if cfg["solve"] in ("bi", "both"):
            t = time.time()
            dlo = Disc(cfg["centers"], cfg["p_lo"], cfg["radius"], cfg["mu"])
            A_lo = lambda v: lcp.lcp_mvp(dlo, pairs, nrm, v, tol=GMRES_TOL)
            x, rep = pqn.bi_pqn(A_hi, A_lo, b, np.zeros(len(pairs)), eps_abs=EPS_KKT)
            times["bi"] = time.time() - t
            out.update(lam_bi=x, bi_iters=rep["iterations"], bi_hi_mvps=rep["hi_mvps"],
                       bi_lo_mvps=rep["lo_mvps"], bi_kkt=rep["kkt_abs"], bi_term=rep["termination"],
                       p_lo=cfg["p_lo"])
            log("c%d bi-PQN iters %d hi %d lo %d kkt %.2e %.1fs" % (c, rep["iterations"], rep["hi_mvps"],
                                                                  rep["lo_mvps"], rep["kkt_abs"], times["bi"]))
    out["times_json"] = repr(times)
    out["total_s"] = time.time() - t0
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "c%d.npz" % c)
    np.savez_compressed(path, **out)
    log("wrote", path, "%.1fs" % out["total_s"])


def run_dense(c):
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "c%d.npz" % c)
    out = dict(np.load(path, allow_pickle=True))
    cfg = make_config(c)
    pairs, nrm = out["pairs"], out["normals"]
    b = out["b"]
    nc = len(pairs)
    times = {}
    t = time.time()
    d = Disc(cfg["centers"], cfg["p"], cfg["radius"], cfg["mu"])
    A = lcp.densify(lambda v: lcp.lcp_mvp(d, pairs, nrm, v, tol=GMRES_TOL), nc)
    times["densify_hi"] = time.time() - t
    log("c%d dense A (%d MVPs) %.1fs" % (c, nc, times["densify_hi"]))
    out.update(A_dense=A)
    if cfg["solve"] in ("mono", "both"):
        t = time.time()
        x, g, _, _, rep = pqn.mono_pqn(lambda v: (A @ v, None), b, np.zeros(nc), eps_abs=EPS_KKT)
        times["mono_dense"] = time.time() - t
        out.update(lam_mono=x, mono_iters=rep["iterations"], mono_mvps=rep["mvps"],
                   mono_kkt=rep["kkt_abs"], mono_term=rep["termination"])
        log("c%d mono-PQN (dense) iters %d mvps %d kkt %.2e" % (c, rep["iterations"], rep["mvps"],
                                                                 rep["kkt_abs"]))
    if cfg["solve"] in ("bi", "both"):
        t = time.time()
        dlo = Disc(cfg["centers"], cfg["p_lo"], cfg["radius"], cfg["mu"])
        Alo = lcp.densify(lambda v: lcp.lcp_mvp(dlo, pairs, nrm, v, tol=GMRES_TOL), nc)
        times["densify_lo"] = time.time() - t
        x, rep = pqn.bi_pqn(lambda v: A @ v, lambda v: Alo @ v, b, np.zeros(nc), eps_abs=EPS_KKT)
        out.update(A_lo_dense=Alo, lam_bi=x, bi_iters=rep["iterations"], bi_hi_mvps=rep["hi_mvps"],
                   bi_lo_mvps=rep["lo_mvps"], bi_kkt=rep["kkt_abs"], bi_term=rep["termination"],
                   p_lo=cfg["p_lo"])
        log("c%d bi-PQN (dense, R34) iters %d hi %d lo %d kkt %.2e" % (c, rep["iterations"], rep["hi_mvps"],
                                                                      rep["lo_mvps"], rep["kkt_abs"]))
    out["dense_times_json"] = repr(times)
    out["dense_cores"] = os.cpu_count()
    np.savez_compressed(path, **out)
    log("wrote", path)


def run_certify(c, lam_path):
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "c%d.npz" % c)
    cfg = make_config(c)
    t = time.time()
    d = Disc(cfg["centers"], cfg["p"], cfg["radius"], cfg["mu"])
    d.near_T_all(workers=os.cpu_count() or 1)
    d.self_full()
    t_pre = time.time() - t
    log("c%d oracle operator data built %.1fs; waiting for %s" % (c, t_pre, lam_path))
    while not os.path.exists(lam_path):
        time.sleep(30)
    time.sleep(5)
    lam = np.load(lam_path)
    out = dict(np.load(path, allow_pickle=True))
    assert lam.shape == (len(out["pairs"]),) and (lam >= 0).all()
    t = time.time()
    w, info = lcp.lcp_mvp(d, out["pairs"], out["normals"], lam, tol=GMRES_TOL, return_info=True)
    t_mvp = time.time() - t
    kkt = float(np.linalg.norm(np.minimum(lam, w + out["b"])))
    h = np.array(info["hist"])
    out["oracle_kg_1e-8"] = int(np.argmax(h <= 1e-8)) + 1 if (h <= 1e-8).any() else -1
    out["oracle_gmres_hist"] = h
    log("c%d certificate: oracle MVP %.1fs (%d its), ||min(lam, A lam + b)|| = %.3e" % (c, t_mvp, info["iters"], kkt))
    out.update(lam_cert=lam, A_lam_cert=w, cert_kkt=kkt, cert_times_json=repr(dict(precompute=t_pre, mvp=t_mvp)),
               cert_cores=os.cpu_count())
    np.savez_compressed(path, **out)
    log("wrote", path)


if __name__ == "__main__":
    if "--certify" in sys.argv:
        native.build()
        a = [x for x in sys.argv[1:] if not x.startswith("--")]
        run_certify(int(a[0]), a[1])
        sys.exit(0)
    if "--dense" in sys.argv:
        native.build()
        for c in [int(a) for a in sys.argv[1:] if not a.startswith("--")]:
            run_dense(c)
        sys.exit(0)
    native.build()
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    cs = [int(a) for a in args] or [1, 2, 3, 4]
    for c in cs:
        run(c, do_lcp=("--no-lcp" not in sys.argv) and c != 4)
