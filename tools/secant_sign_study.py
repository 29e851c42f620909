"""Reading R34 study: Bi-PQN (oracle, Alg. 3) lo/hi MVP counts with the re-used secants
transformed by the paper's requirement (Y^ + (uu^T - vv^T) S^) versus the
printed display (Y^ - (uu^T - vv^T) S^), on seeded dense LCPs."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import pqn  # noqa: E402


def lcp(seed, n):
    rng = np.random.default_rng(seed)
    M = rng.standard_normal((n, n))
    A = M @ M.T / n + 0.05 * np.eye(n)
    E = rng.standard_normal((n, n)) * 0.1 / np.sqrt(n)
    Ahat = A + E + E.T
    Ahat += max(0.0, 0.02 - np.linalg.eigvalsh(Ahat).min()) * np.eye(n)
    return A, Ahat, rng.standard_normal(n)


def run(sign, n=80, cases=20):
    orig = pqn.transform_secants
    if sign < 0:
        pqn.transform_secants = lambda S, Y, u, v: [y - u * (u @ s) + v * (v @ s) for s, y in zip(S, Y)]
    hi = lo = 0
    try:
        for c in range(cases):
            A, Ahat, b = lcp(1000 + c, n)
            x, rep = pqn.bi_pqn(lambda v: A @ v, lambda v: Ahat @ v, b, np.zeros(n), eps_abs=1e-10)
            assert rep["termination"] == 0
            hi += rep["hi_mvps"]
            lo += rep["lo_mvps"]
    finally:
        pqn.transform_secants = orig
    return hi, lo


if __name__ == "__main__":
    for sign, name in [(-1, "printed (P:486)"), (1, "R34 (B^(k+1) S = Y)")]:
        hi, lo = run(sign)
        print("%-22s hi MVPs %5d  lo MVPs %6d  (20 dense LCPs, n = 80)" % (name, hi, lo))
