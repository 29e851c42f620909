"""Contacts, the contact Jacobian D, the LCP MVP and b (oracle; TEST INFRASTRUCTURE ONLY).

PAPER.md P:152-157 (gap Phi, active set {Phi_l <= delta}), P:166 (F_c = D x, 6 nnz
per column for spheres), P:181 (D^T = grad Phi G), P:182-191 (LCP, A = D^T M D,
b = (Phi + dt D^T U_nc)/dt).  Readings R14 (dt = 1), R20 (strict gap < delta,
lexicographic i < j), O8-O10.

Column l of D: -n_l in sphere i's force rows, +n_l in sphere j's force rows, zero
torque rows, n_l = (c_j - c_i)/|c_j - c_i|.
Pins (tests/test_oracle_operator.py::test_contacts_and_D, test_lcp_matrix_pd_near_contact;
tests/test_oracle_pqn.py brute-force LCPs): D column = finite difference of Phi; D^T of a
common translation = 0; A = D^T M D symmetric / PSD to a p-dependent tolerance
(R27); brute-force active-set enumeration (O14) agrees with the PQN solvers.
"""
import itertools

import numpy as np

from .mobility import mobility


def contacts(centers, a, delta):
    """Returns pairs [Nc,2] (i<j, lexicographic), normals [Nc,3], gaps [Nc]."""
    centers = np.asarray(centers, dtype=np.float64).reshape(-1, 3)
    pairs, normals, gaps = [], [], []
    n = centers.shape[0]
    for i in range(n):
        for j in range(i + 1, n):
            d = centers[j] - centers[i]
            dist = np.linalg.norm(d)
            gap = dist - 2.0 * a
            if gap < delta:
                pairs.append((i, j))
                normals.append(d / dist)
                gaps.append(gap)
    return (np.array(pairs, dtype=np.int64).reshape(-1, 2), np.array(normals).reshape(-1, 3),
            np.array(gaps))


def D_apply(np_, pairs, normals, lam):
    """F_c = D lambda as [Np,6] (torques zero)."""
    FT = np.zeros((np_, 6))
    for l, (i, j) in enumerate(pairs):
        FT[i, :3] -= lam[l] * normals[l]
        FT[j, :3] += lam[l] * normals[l]
    return FT


def DT_apply(pairs, normals, UO):
    """w = D^T (U, Omega): w_l = n_l . (U_j - U_i)."""
    UO = np.asarray(UO).reshape(-1, 6)
    return np.array([np.dot(normals[l], UO[j, :3] - UO[i, :3]) for l, (i, j) in enumerate(pairs)])


def lcp_mvp(disc, pairs, normals, lam, tol=1e-13, return_info=False):
    """w = D^T M D lambda."""
    FT = D_apply(disc.np, pairs, normals, np.asarray(lam, dtype=np.float64))
    UO, info = mobility(disc, FT, None, tol=tol, return_info=True)
    w = DT_apply(pairs, normals, UO)
    return (w, info) if return_info else w


def lcp_b(disc, pairs, normals, gaps, F_nc, slip, dt=1.0, tol=1e-13):
    """b = (Phi + dt D^T U_nc)/dt with U_nc = M_slip(F_nc, 0; u_s) (R14)."""
    FT = np.zeros((disc.np, 6))
    FT[:, :3] = np.asarray(F_nc).reshape(-1, 3)
    U_nc = mobility(disc, FT, slip, tol=tol)
    return (np.asarray(gaps) + dt * DT_apply(pairs, normals, U_nc)) / dt, U_nc


def densify(apply, n):
    """Dense matrix of a linear operator by applying it to unit vectors."""
    cols = []
    for l in range(n):
        e = np.zeros(n)
        e[l] = 1.0
        cols.append(apply(e))
    return np.stack(cols, axis=1)


def brute_force_lcp(A, b, tie=1e-12):
    """O14: enumerate every active set S; accept lambda_S = -A_SS^{-1} b_S when
    lambda_S >= 0 and (A lambda + b)_{S^c} >= 0.  Returns (lambda, number accepted)."""
    n = b.size
    scale = max(1.0, np.abs(b).max())
    found = []
    for mask in itertools.product([False, True], repeat=n):
        S = np.array(mask, dtype=bool)
        lam = np.zeros(n)
        if S.any():
            try:
                lam[S] = np.linalg.solve(A[np.ix_(S, S)], -b[S])
            except np.linalg.LinAlgError:
                continue
        if (lam[S] < -tie * scale).any():
            continue
        wv = A @ lam + b
        if (wv[~S] < -tie * scale).any():
            continue
        found.append(lam)
    if not found:
        return None, 0
    return found[0], len(found)
