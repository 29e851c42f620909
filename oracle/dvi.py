"""One DVI time step (oracle; TEST INFRASTRUCTURE ONLY).

PAPER.md P:140-176: configuration dynamics dC/dt = G U_nc + G M F_c (eq. dynamSys),
forward Euler C^{i+1} = C^i + dt (G U_nc + G M D x) with 0 <= Phi_A(C^{i+1}) _|_ x >= 0
linearised into the LCP 0 <= A x + b _|_ x >= 0, A = D^T M D, b = (Phi + dt D^T U_nc)/dt
(P:182-188).  Orientation (reading R32): the Janus axis of each sphere is advanced by
a <- normalise(a + dt Omega x a) (first-order rotation; quaternions are out of scope).
Pins (tests/test_oracle_dvi.py): no contacts -> the free mobility step; a pushed-together
pair ends the step with linearised gap exactly 0 and lambda > 0; a free Janus sphere
swims along its axis.
"""
import numpy as np

from . import lcp
from . import mobility as mob
from . import pqn
from .layer import Disc


def solve_lcp_exact(A_apply, b, nc):
    """The unique LCP solution: brute force for nc <= 12 (O14), else Mono-PQN to 1e-12."""
    if nc <= 12:
        A = lcp.densify(A_apply, nc)
        lam, cnt = lcp.brute_force_lcp(A, b)
        assert cnt >= 1
        return lam
    x, g, _, _, rep = pqn.mono_pqn(lambda v: (A_apply(v), None), b, np.zeros(nc), eps_abs=1e-12)
    return x


def dvi_step(centers, axes, F_nc, p, dt, delta=0.1, slip_B=1.0, a=1.0, mu=1.0, tol=1e-13):
    """Returns (new_centers, new_axes, UO [Np,6], lam, pairs)."""
    centers = np.asarray(centers, dtype=np.float64).reshape(-1, 3)
    axes = np.asarray(axes, dtype=np.float64).reshape(-1, 3)
    d = Disc(centers, p, a, mu)
    pairs, nrm, gaps = lcp.contacts(centers, a, delta)
    slip = mob.janus_slip(d, axes, slip_B)
    FT = np.zeros((d.np, 6))
    FT[:, :3] = np.asarray(F_nc).reshape(-1, 3)
    U_nc = mob.mobility(d, FT, slip, tol=tol)
    U = U_nc.copy()
    lam = np.zeros(len(pairs))
    if len(pairs):
        b = (gaps + dt * lcp.DT_apply(pairs, nrm, U_nc)) / dt
        A_apply = lambda v: lcp.lcp_mvp(d, pairs, nrm, v, tol=tol)
        lam = solve_lcp_exact(A_apply, b, len(pairs))
        U = U + mob.mobility(d, lcp.D_apply(d.np, pairs, nrm, lam), None, tol=tol)
    new_c = centers + dt * U[:, :3]
    new_a = axes + dt * np.cross(U[:, 3:], axes)
    new_a /= np.linalg.norm(new_a, axis=1, keepdims=True)
    return new_c, new_a, U, lam, pairs
