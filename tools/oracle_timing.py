"""Whole-oracle timings on the host cores of the GPU box (SURVEY 8(d) "Oracle timing"): one oracle LCP
MVP at c1-c3 (GMRES 1e-8, the oracle's own iteration count from its residual history), full oracle
Mono-PQN solves at c1-c2 (paper mode: GMRES 1e-8, KKT 1e-8), and bench.py's per-pass sample model at
the same k_g beside each measured MVP (validates the extrapolation bench.py uses for c4).
Geometry precompute (near tensors, self rows) is timed separately, like bpqn_geometry_init.
  python tools/oracle_timing.py [--solve-c2] [--solve-c3] > profiles/r02_oracle_timing.jsonl"""
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from oracle import lcp, native, pqn  # noqa: E402
from oracle.layer import Disc  # noqa: E402
from synth import lambda_test, make_config  # noqa: E402

native.build()
print(json.dumps({"host": bench.cpu_desc(), "cores": os.cpu_count(), "omp": os.environ.get("OMP_NUM_THREADS"),
                  "python": platform.python_version()}), flush=True)
for c in (1, 2, 3):
    cfg = make_config(c)
    t = time.perf_counter()
    d = Disc(cfg["centers"], cfg["p"], cfg["radius"], cfg["mu"])
    d.near_T_all(workers=os.cpu_count() or 1)
    d.self_full()
    t_pre = time.perf_counter() - t
    pairs, nrm, gaps = lcp.contacts(cfg["centers"], cfg["radius"], cfg["delta"])
    lam = lambda_test(c, len(pairs), 0)
    t = time.perf_counter()
    w, info = lcp.lcp_mvp(d, pairs, nrm, lam, tol=1e-8, return_info=True)
    t_mvp = time.perf_counter() - t
    model = bench.oracle_mvp_sample(cfg, info["iters"])
    print(json.dumps({"config": c, "N": d.N, "precompute_s": round(t_pre, 2), "mvp_s": round(t_mvp, 3),
                      "gmres_iters": info["iters"], "model_mvp_s": round(model["ms"] / 1e3, 3),
                      "model_per_pass_s": model["per_pass_s"]}), flush=True)
    if c == 1 or (c == 2 and "--solve-c2" in sys.argv) or (c == 3 and "--solve-c3" in sys.argv):
        from oracle import mobility as mob
        slip = mob.janus_slip(d, cfg["axes"], cfg["slip_B"])
        t = time.perf_counter()
        b, _ = lcp.lcp_b(d, pairs, nrm, gaps, cfg["F_nc"], slip, tol=1e-8)
        t_b = time.perf_counter() - t
        A_hi = lambda v: lcp.lcp_mvp(d, pairs, nrm, v, tol=1e-8)  # noqa: E731
        if c in (1, 2):
            t = time.perf_counter()
            x, g, _, _, rep = pqn.mono_pqn(lambda v: (A_hi(v), None), b, np.zeros(len(pairs)), eps_abs=1e-8,
                                           eps_rel=1e-8)
            print(json.dumps({"config": c, "solve": "Mono-PQN (paper mode)", "b_s": round(t_b, 2),
                              "solve_s": round(time.perf_counter() - t, 2), "mvps": rep["mvps"],
                              "iterations": rep["iterations"], "kkt": rep["kkt_abs"]}), flush=True)
        if c in (2, 3) and cfg.get("p_lo"):
            t = time.perf_counter()
            dlo = Disc(cfg["centers"], cfg["p_lo"], cfg["radius"], cfg["mu"])
            dlo.near_T_all(workers=os.cpu_count() or 1)
            dlo.self_full()
            t_pre = time.perf_counter() - t
            A_lo = lambda v: lcp.lcp_mvp(dlo, pairs, nrm, v, tol=1e-6)  # noqa: E731  (R36: lo eps 1e-6)
            t = time.perf_counter()
            x, rep = pqn.bi_pqn(A_hi, A_lo, b, np.zeros(len(pairs)), eps_abs=1e-8, eps_rel=1e-8)
            print(json.dumps({"config": c, "solve": "Bi-PQN (paper mode, matrix-free lo)", "b_s": round(t_b, 2),
                              "lo_precompute_s": round(t_pre, 2), "solve_s": round(time.perf_counter() - t, 2),
                              "hi_mvps": rep["hi_mvps"], "lo_mvps": rep["lo_mvps"],
                              "iterations": rep["iterations"], "kkt": rep["kkt_abs"]}), flush=True)
