"""Preconditioner study on the dense completed double-layer operator (bpqn_operator_dense), torch on the GPU
(development aid): right-preconditioned GMRES iterations to 1e-8 for the mobility right-hand side of a seeded
force set, with no preconditioner, the library's per-sphere block-Jacobi, and block-Jacobi over clusters of
spheres (spatial cells of cell x cell x cell lattice sites).
  python tools/precond_study.py --config 4 --p 8 [--sub 3] [--cells 2,3]"""
import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_10089_b200 as bp  # noqa: E402
from synth import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--p", type=int, default=8)
ap.add_argument("--sub", type=int, default=0)      # keep the spheres of a sub x sub x sub corner of the lattice
ap.add_argument("--cells", default="2,3")
ap.add_argument("--tol", type=float, default=1e-8)
ap.add_argument("--coarse", default="1,2")   # two-level: per-sphere polynomial coarse spaces of these degrees
a = ap.parse_args()
cfg = make_config(a.config)
C = cfg["centers"]
if a.sub:
    lo = C.min(axis=0)
    keep = np.all(C - lo < a.sub * 2.02 - 0.5, axis=1)
    C = C[keep]
g = bp.Geometry(C, a.p)
n = 3 * g.N
t = time.time()
A = bp._bpqn.operator_dense(g)
torch.cuda.synchronize()
t_asm = time.time() - t
rng = np.random.default_rng(5)
F = rng.standard_normal((g.np, 3))
f = torch.tensor(np.repeat(F / (4 * math.pi), g.nq, axis=0), device="cuda")
rhs = -bp.layer_apply(g, f, None).reshape(-1)
nqv = 3 * g.nq


def gmres(apply_prec, tol, m=300):
    beta = torch.linalg.norm(rhs)
    V = torch.zeros((m + 1, n), dtype=torch.float64, device="cuda")
    H = torch.zeros((m + 1, m), dtype=torch.float64, device="cuda")
    V[0] = rhs / beta
    e1 = torch.zeros(m + 1, dtype=torch.float64, device="cuda")
    e1[0] = beta
    for k in range(m):
        w = A @ apply_prec(V[k])
        for _ in range(2):
            h = V[: k + 1] @ w
            w = w - V[: k + 1].T @ h
            H[: k + 1, k] += h
        H[k + 1, k] = torch.linalg.norm(w)
        V[k + 1] = w / H[k + 1, k]
        y = torch.linalg.lstsq(H[: k + 2, : k + 1], e1[: k + 2, None]).solution
        res = torch.linalg.norm(e1[: k + 2] - H[: k + 2, : k + 1] @ y[:, 0]) / beta
        if res <= tol:
            return k + 1
    return m


def block_inv(groups):
    """inverses of the diagonal blocks of A over groups of spheres (lists of sphere indices)"""
    out = []
    for grp in groups:
        idx = torch.cat([torch.arange(s * nqv, (s + 1) * nqv, device="cuda") for s in grp])
        out.append((idx, torch.linalg.inv(A[idx][:, idx])))
    return out


def prec_of(blocks):
    def ap(v):
        z = torch.empty_like(v)
        for idx, Bi in blocks:
            z[idx] = Bi @ v[idx]
        return z
    return ap


res = dict(config=a.config, p=a.p, spheres=g.np, N=g.N, assemble_s=round(t_asm, 2))
res["none"] = gmres(lambda v: v, a.tol)
res["sphere_bj"] = gmres(prec_of(block_inv([[s] for s in range(g.np)])), a.tol)
cen = C - C.min(axis=0)
for cell in [int(x) for x in a.cells.split(",") if x]:
    key = np.floor(cen / (cell * 2.02 - 1e-6)).astype(int)
    groups = {}
    for s, k in enumerate(map(tuple, key)):
        groups.setdefault(k, []).append(s)
    t = time.time()
    blocks = block_inv(list(groups.values()))
    res["cluster%d_bj" % cell] = gmres(prec_of(blocks), a.tol)
    res["cluster%d_setup_s" % cell] = round(time.time() - t, 2)
    res["cluster%d_blocks" % cell] = len(groups)
    del blocks
    torch.cuda.empty_cache()
# two-level additive preconditioner: sphere block-Jacobi + Galerkin coarse correction on per-sphere
# polynomial fields of degree <= L in the unit normal (x 3 components), orthonormalised per sphere
t_, w_ = np.polynomial.legendre.leggauss(a.p + 1)
t_ = t_[::-1]
th = np.arccos(t_)
ph = np.pi * np.arange(2 * a.p) / a.p
xi = np.stack([np.outer(np.sin(th), np.cos(ph)).ravel(), np.outer(np.sin(th), np.sin(ph)).ravel(),
               np.repeat(np.cos(th), 2 * a.p)], axis=1)
bj = prec_of(block_inv([[s] for s in range(g.np)]))
for L in [int(x) for x in a.coarse.split(",") if x]:
    mons = [np.ones(len(xi))]
    for d in range(1, L + 1):
        for i in range(d + 1):
            for j in range(d + 1 - i):
                k = d - i - j
                mons.append(xi[:, 0] ** i * xi[:, 1] ** j * xi[:, 2] ** k)
    P = np.stack(mons, axis=1)                      # [nq, nm]
    Q, _ = np.linalg.qr(P)
    nm = Q.shape[1]
    local = np.zeros((3 * g.nq, 3 * nm))
    for c in range(3):
        local[c::3, c::3] = Q                        # component c of node j is entry 3 j + c
    Zl = torch.tensor(local, device="cuda")
    Z = torch.zeros((n, g.np * 3 * nm), dtype=torch.float64, device="cuda")
    for s_ in range(g.np):
        Z[s_ * nqv:(s_ + 1) * nqv, s_ * 3 * nm:(s_ + 1) * 3 * nm] = Zl
    E = Z.T @ (A @ Z)
    Einv = torch.linalg.inv(E)

    def two_level(v, Z=Z, Einv=Einv):
        return bj(v) + Z @ (Einv @ (Z.T @ v))
    res["two_level_deg%d" % L] = gmres(two_level, a.tol)
    res["two_level_deg%d_coarse_dim" % L] = int(Z.shape[1])
    del Z, E, Einv
    torch.cuda.empty_cache()
print(json.dumps(res), flush=True)
