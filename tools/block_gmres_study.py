"""Block GMRES study for forming the low-fidelity LCP matrix (R38), torch on the GPU (development aid).
The Nc right-hand sides -S[P^T D e_l] of one A^ formation share the operator's slow modes, so one block
Krylov space (dimension Nc per iteration) should need far fewer operator applications than Nc independent
GMRES processes (the library's batched GMRES: 42 iterations at c4 lo, 1e-6).  Dense operator from
bpqn_operator_dense, right block-Jacobi (per-sphere self block inverse), block CGS2, Cholesky-QR2 of each
block, least squares of the block Hessenberg per iteration (torch.linalg.lstsq).
  python tools/block_gmres_study.py --config 4 --p 8 --tol 1e-6"""
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
ap.add_argument("--tol", type=float, default=1e-6)
ap.add_argument("--maxit", type=int, default=40)
ap.add_argument("--ncols", type=int, default=0)
a = ap.parse_args()
cfg = make_config(a.config)
g = bp.Geometry(cfg["centers"], a.p)
pairs, nrm, gaps = bp.contacts(g, 0.1)
nc = g.nc if a.ncols == 0 else min(a.ncols, g.nc)
n = 3 * g.N
nqv = 3 * g.nq
t = time.time()
A = bp._bpqn.operator_dense(g)
torch.cuda.synchronize()
print("operator", A.shape, "%.2f s" % (time.time() - t), flush=True)
# right-hand sides -S[P^T D e_l]: contact forces -n on sphere i, +n on sphere j, no torque
xi = None
pr, nm = pairs.cpu().numpy(), nrm.cpu().numpy()
B = torch.empty((n, nc), dtype=torch.float64, device="cuda")
for l in range(nc):
    F = np.zeros((g.np, 3))
    F[pr[l, 0]] -= nm[l]
    F[pr[l, 1]] += nm[l]
    f = torch.tensor(np.repeat(F / (4 * math.pi), g.nq, axis=0), device="cuda")
    B[:, l] = -bp.layer_apply(g, f, None).reshape(-1)
bn = torch.linalg.norm(B, dim=0)
E = A[:nqv, :nqv]
Einv = torch.linalg.inv(E.clone())


def prec(X):  # right block-Jacobi: per-sphere self-block inverse
    Y = X.reshape(g.np, nqv, -1)
    return torch.einsum("ij,sjk->sik", Einv, Y).reshape(n, -1)


def cholqr2(W):
    R = torch.eye(W.shape[1], dtype=W.dtype, device=W.device)
    for _ in range(2):
        G = W.T @ W
        L = torch.linalg.cholesky(G)
        W = torch.linalg.solve_triangular(L, W.T, upper=False).T
        R = L.T @ R
    return W, R


def batched_gmres_iters():
    """the library's scheme for reference: Nc independent GMRES processes (iterations until all converge)"""
    return None


t0 = time.time()
V0, S0 = cholqr2(B.clone())
Vs = [V0]
Hcols = []   # H[:, k] blocks: list of lists
res_hist = []
m = nc
for k in range(a.maxit):
    W = A @ prec(Vs[k])
    hk = []
    for _ in range(2):
        Vall = torch.cat(Vs, dim=1)
        h = Vall.T @ W
        W = W - Vall @ h
        hk.append(h)
    h = hk[0] + hk[1]
    Vn, Rn = cholqr2(W)
    Vs.append(Vn)
    col = torch.zeros(((k + 2) * m, m), dtype=torch.float64, device="cuda")
    col[: (k + 1) * m] = h
    col[(k + 1) * m:] = Rn
    Hcols.append(col)
    Hbar = torch.zeros(((k + 2) * m, (k + 1) * m), dtype=torch.float64, device="cuda")
    for j, c in enumerate(Hcols):
        Hbar[: c.shape[0], j * m:(j + 1) * m] = c
    rhs = torch.zeros(((k + 2) * m, m), dtype=torch.float64, device="cuda")
    rhs[:m] = S0
    Y = torch.linalg.lstsq(Hbar, rhs).solution
    R = rhs - Hbar @ Y
    rel = torch.linalg.norm(R, dim=0) / bn
    torch.cuda.synchronize()
    res_hist.append(float(rel.max()))
    print("block it %d max rel res %.3e median %.3e  %.1f s" % (k + 1, rel.max(), rel.median(), time.time() - t0),
          flush=True)
    if rel.max() <= a.tol:
        break
# true residual check
X = prec(torch.cat(Vs[:-1], dim=1) @ Y)
tr = torch.linalg.norm(B - A @ X, dim=0) / bn
print(json.dumps({"config": a.config, "p": a.p, "nc": nc, "n": n, "tol": a.tol, "block_iterations": len(res_hist),
                  "true_rel_res_max": float(tr.max()), "res_hist": res_hist, "wall_s": time.time() - t0}))
