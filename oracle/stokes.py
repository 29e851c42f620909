"""Free-space Stokes kernels and the singular self quadrature (oracle; TEST INFRASTRUCTURE ONLY).

Kernels (reading R3, O3; PAPER.md P:53-69 gives the PDE, P:130-134 the operator
M^stk, neither gives a discretisation).  With r = x - y, rho = |r|:

    G(r)      = 1/(8 pi mu) * (I/rho + r r^T / rho^3)              (Stokeslet)
    K_D(x, y) = -3/(4 pi) * (r . n_y) r r^T / rho^5                 (stresslet)

Self quadrature (reading R5/R6, O3): for target node i at (theta_i, phi_i) rotate
a Gauss-Legendre(theta' on [0, pi]) x trapezoid(phi') grid of order p_s by
R_i = R_z(phi_i) R_y(theta_i) so that its pole sits on the target, and integrate
kernel * (Pi_p interpolant of the density) there:

    S_self[i, j] = sum_s w'_s G(x_i - y'_s) Pi_j(y'_s),
    w'_s = a^2 sin(theta'_k) (pi/2) omega'_k (pi/p_s).

Pins (tests/test_oracle_geometry.py: test_self_closed_forms, test_self_converged_in_ps): closed forms on a sphere (App. A.1):
S[const] = 2a/(3 mu) const (Stokes drag), S[rotation traction] = Omega x x,
S[xi] = 0; Gauss identity D[const] = const/2, rigid motions eigenvalue +1/2, the
normal field eigenvalue -1/2; both to <= 1e-10 at the configs' p.
"""
import numpy as np

from .grid import gauss_legendre


def stokeslet(r, mu):
    """G(r) for r [..., 3] -> [..., 3, 3]."""
    rho2 = np.sum(r * r, axis=-1)
    rho = np.sqrt(rho2)
    eye = np.eye(3)
    return (eye / rho[..., None, None] + r[..., :, None] * r[..., None, :] / (rho ** 3)[..., None, None]) / (8.0 * np.pi * mu)


def stresslet(r, n):
    """K_D for r = x - y [..., 3] and source normal n [..., 3] -> [..., 3, 3]."""
    rho2 = np.sum(r * r, axis=-1)
    rho = np.sqrt(rho2)
    rn = np.sum(r * n, axis=-1)
    return -3.0 / (4.0 * np.pi) * (rn / rho ** 5)[..., None, None] * r[..., :, None] * r[..., None, :]


def rot_y(t):
    c, s = np.cos(t), np.sin(t)
    return np.array([[c, 0.0, s], [0.0, 1.0, 0.0], [-s, 0.0, c]])


def rot_z(t):
    c, s = np.cos(t), np.sin(t)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


def singular_grid(ps):
    """Unit points eta [n_s, 3] and unit-sphere weights [n_s] of the polar grid of
    order ps: Gauss-Legendre in theta' on [0, pi] (ps+1 nodes) x 2ps phi'."""
    t, om = gauss_legendre(ps + 1)
    thp = 0.5 * np.pi * (t + 1.0)
    wth = 0.5 * np.pi * om * np.sin(thp)
    php = np.pi * np.arange(2 * ps) / ps
    th, ph = np.meshgrid(thp, php, indexing="ij")
    st = np.sin(th)
    eta = np.stack([st * np.cos(ph), st * np.sin(ph), np.cos(th)], axis=-1).reshape(-1, 3)
    wts = np.outer(wth, np.full(2 * ps, np.pi / ps)).reshape(-1)
    return eta, wts


def self_rows(grid, proj, i, ps, mu):
    """Rows of S_self and D_self for local target node i (sphere centred at 0).

    Returns (S_row, D_row), each [3, Nq, 3]: u_i[a] = sum_{j,b} row[a, j, b] dens_j[b]."""
    a = grid["a"]
    eta, wts = singular_grid(ps)
    R = rot_z(grid["phi_node"][i]) @ rot_y(grid["theta_node"][i])
    pts = eta @ R.T                       # rotated unit points
    y = a * pts
    x = a * grid["xi"][i]
    r = x[None, :] - y
    wq = a * a * wts
    Pi = proj.interp_rows(pts)            # [n_s, Nq]
    G = stokeslet(r, mu) * wq[:, None, None]
    K = stresslet(r, pts) * wq[:, None, None]
    S_row = np.einsum("sab,sj->ajb", G, Pi)
    D_row = np.einsum("sab,sj->ajb", K, Pi)
    return S_row, D_row


def self_matrices(grid, proj, ps, mu):
    """Full S_self, D_self as [Nq, 3, Nq, 3] (every target computed directly)."""
    nq = grid["xi"].shape[0]
    S = np.zeros((nq, 3, nq, 3))
    D = np.zeros((nq, 3, nq, 3))
    for i in range(nq):
        S[i], D[i] = self_rows(grid, proj, i, ps, mu)
    return S, D
