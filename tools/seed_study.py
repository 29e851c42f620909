"""Does the Krylov space of some right-hand sides help others? (development aid for R38's batched GMRES)
On the dense low-fidelity operator (c4 centres, p = 8) with the per-sphere block-Jacobi preconditioner:
GMRES iterations to 1e-6 for LCP right-hand sides b_l = -S[P^T D e_l] from zero, and from the Galerkin
projection onto the Krylov spaces of a first batch of columns."""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_10089_b200 as bp  # noqa: E402
from synth import make_config  # noqa: E402

cfg = make_config(4)
g = bp.Geometry(cfg["centers"], 8)
pairs, nrm, gaps = bp.contacts(g, cfg["delta"])
n = 3 * g.N
A = bp._bpqn.operator_dense(g)
nqv = 3 * g.nq
Binv = []
for s in range(g.np):
    sl = slice(s * nqv, (s + 1) * nqv)
    Binv.append(torch.linalg.inv(A[sl, sl]))
Binv = torch.stack(Binv)                         # [np, nqv, nqv]


def prec(v):                                     # v [n, k]
    return torch.einsum("sij,sjk->sik", Binv, v.reshape(g.np, nqv, -1)).reshape(n, -1)


P = pairs.cpu().numpy()
Nn = nrm.cpu().numpy()
rng = np.random.default_rng(1)


def rhs(l):
    i, j = P[l]
    F = np.zeros((g.np, 3))
    F[i] -= Nn[l]
    F[j] += Nn[l]
    f = torch.tensor(np.repeat(F / (4 * math.pi), g.nq, axis=0), device="cuda")
    return -bp.layer_apply(g, f, None).reshape(-1)


def gmres(b, x0=None, tol=1e-6, m=200, keep=None):
    r = b - (A @ x0 if x0 is not None else 0)
    beta0 = torch.linalg.norm(b)
    beta = torch.linalg.norm(r)
    V = torch.zeros((m + 1, n), dtype=torch.float64, device="cuda")
    Z = torch.zeros((m, n), dtype=torch.float64, device="cuda")
    H = torch.zeros((m + 1, m), dtype=torch.float64, device="cuda")
    V[0] = r / beta
    e1 = torch.zeros(m + 1, dtype=torch.float64, device="cuda")
    e1[0] = beta
    if beta / beta0 <= tol:
        return 0, float(beta / beta0)
    for k in range(m):
        Z[k] = prec(V[k:k + 1].T)[:, 0]
        w = A @ Z[k]
        for _ in range(2):
            h = V[: k + 1] @ w
            w = w - V[: k + 1].T @ h
            H[: k + 1, k] += h
        H[k + 1, k] = torch.linalg.norm(w)
        V[k + 1] = w / H[k + 1, k]
        y = torch.linalg.lstsq(H[: k + 2, : k + 1], e1[: k + 2, None]).solution
        res = torch.linalg.norm(e1[: k + 2] - H[: k + 2, : k + 1] @ y[:, 0]) / beta0
        if res <= tol:
            if keep is not None:
                keep.append(Z[: k + 1].clone())
            return k + 1, float(beta / beta0)
    return m, float(beta / beta0)


cols = rng.permutation(len(P))
first, second = cols[:48], cols[48:96]
basis = []
it_first = [gmres(rhs(l), keep=basis)[0] for l in first]
Zs = torch.cat(basis)                            # search directions of the first batch (x lives in their span)
AZ = A @ Zs.T                                    # [n, K]
Q, R = torch.linalg.qr(AZ)
res = dict(first_batch=len(first), first_mean_its=float(np.mean(it_first)), span_dim=int(Zs.shape[0]))
cold, warm, r0 = [], [], []
for l in second:
    b = rhs(l)
    cold.append(gmres(b)[0])
    c = torch.linalg.solve_triangular(R, (Q.T @ b)[:, None], upper=True)[:, 0]   # min |A Z c - b|
    x0 = Zs.T @ c
    k, rr = gmres(b, x0=x0)
    warm.append(k)
    r0.append(rr)
res.update(second_cold_mean_its=float(np.mean(cold)), second_warm_mean_its=float(np.mean(warm)),
           second_warm_initial_resid_median=float(np.median(r0)))
print(json.dumps(res), flush=True)
