"""Real spherical harmonics and the order-p projection Pi_p (oracle; TEST INFRASTRUCTURE ONLY).

Reading R7 / O2: "order-p spherical harmonics" is
read as V_p = span{real Y_lm : l <= p} minus the sectoral sin(p phi) function
(identically zero on the phi grid), dim V_p = p^2 + 2p.  The interpolant of nodal
values at any point is their quadrature-weighted least-squares projection onto V_p,
evaluated at that point.  The oracle writes that definition out literally:

    Pi(Z) = Y(Z) (Y^T W Y)^{-1} Y^T W            (Y = basis at the grid nodes)

with a dense solve -- it does NOT use the closed-form "halve the cos(p phi)
coefficient" shortcut the CUDA path uses (App. A.3), so agreement of the two is a
check of that derivation.

Pins (tests/test_oracle_geometry.py: test_legendre_vs_scipy,
test_legendre_recurrence_small_closed_forms, test_sh_orthonormal_and_nyquist, test_projection): the Legendre recurrence against
scipy.special.sph_harm_y; orthonormality under exact (high-order) quadrature;
Pi reproduces V_p and is idempotent; Pi annihilates sin(p phi) P_p^p.
"""
import numpy as np


def basis_lm(p):
    """(l, m) list for V_p: l = 0..p, m = -l..l, without (p, -p) (sin p phi)."""
    out = []
    for l in range(p + 1):
        for m in range(-l, l + 1):
            if l == p and m == -p:
                continue
            out.append((l, m))
    return out


def norm_legendre(lmax, t):
    """Fully normalised associated Legendre functions Pbar[l][m](t), m >= 0,
    with int_{-1}^{1} Pbar^2 dt = 1 (textbook three-term recurrence).
    Returns array [lmax+1, lmax+1, len(t)] (zero for m > l)."""
    t = np.asarray(t, dtype=np.float64)
    s = np.sqrt(np.maximum(0.0, 1.0 - t * t))
    P = np.zeros((lmax + 1, lmax + 1) + t.shape)
    P[0, 0] = 1.0 / np.sqrt(2.0)
    for m in range(1, lmax + 1):
        P[m, m] = -np.sqrt((2.0 * m + 1.0) / (2.0 * m)) * s * P[m - 1, m - 1]
    for m in range(0, lmax):
        P[m + 1, m] = np.sqrt(2.0 * m + 3.0) * t * P[m, m]
    for m in range(0, lmax + 1):
        for l in range(m + 2, lmax + 1):
            a = np.sqrt((4.0 * l * l - 1.0) / (l * l - m * m))
            b = np.sqrt(((l - 1.0) ** 2 - m * m) / (4.0 * (l - 1.0) ** 2 - 1.0))
            P[l, m] = a * (t * P[l - 1, m] - b * P[l - 2, m])
    return P


def real_sh(p, xyz):
    """Orthonormal (on the unit sphere) real SH of V_p at unit vectors xyz [n,3].
    Returns [n, nb] with columns ordered as basis_lm(p)."""
    xyz = np.asarray(xyz, dtype=np.float64)
    t = np.clip(xyz[:, 2], -1.0, 1.0)
    phi = np.arctan2(xyz[:, 1], xyz[:, 0])
    P = norm_legendre(p, t)
    cols = []
    for (l, m) in basis_lm(p):
        if m == 0:
            cols.append(P[l, 0] / np.sqrt(2.0 * np.pi))
        elif m > 0:
            cols.append(P[l, m] * np.cos(m * phi) / np.sqrt(np.pi))
        else:
            cols.append(P[l, -m] * np.sin(-m * phi) / np.sqrt(np.pi))
    return np.stack(cols, axis=1)


class Projector:
    """Weighted least-squares projection onto V_p for the order-p grid (O2)."""

    def __init__(self, grid):
        self.p = grid["p"]
        self.xi = grid["xi"]
        self.w = grid["w"]
        Y = real_sh(self.p, self.xi)              # [Nq, nb]
        WY = Y * self.w[:, None]
        gram = Y.T @ WY                           # Y^T W Y
        # analysis operator: coefficients = gram^{-1} Y^T W f
        self.analysis = np.linalg.solve(gram, WY.T)   # [nb, Nq]
        self.Y = Y

    def interp_rows(self, unit_pts):
        """Rows Pi_j(y) for points y on the unit sphere: [n, Nq]."""
        return real_sh(self.p, unit_pts) @ self.analysis

    def matrix(self):
        """Pi_p on the grid itself: [Nq, Nq]."""
        return self.Y @ self.analysis
