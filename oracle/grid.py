"""Sphere quadrature grids (oracle; TEST INFRASTRUCTURE ONLY).

Reading R10 / O1: the paper only states that order-p spherical
harmonics with N = 6 Np p(p+1) dof are used.  Per sphere we use
(p+1) Gauss-Legendre nodes in t = cos(theta) (k = 0 nearest the north pole) times
2p equispaced phi_l = pi l / p, weight w_kl = a^2 omega_k pi / p, local index
i = k*2p + l.  Pinned by tests/test_oracle_geometry.py::test_grid_moments (sphere moments to degree 2p,
sum w = 4 pi a^2).
"""
import numpy as np


def gauss_legendre(n):
    """n-point Gauss-Legendre rule on [-1, 1], nodes in DESCENDING order.

    Library primitive (numpy.polynomial.legendre.leggauss)."""
    t, w = np.polynomial.legendre.leggauss(n)
    order = np.argsort(-t)
    return t[order], w[order]


def sphere_grid(p, a=1.0):
    """Order-p grid on a sphere of radius a centred at the origin.

    Returns dict with theta[p+1], phi[2p], xi[Nq,3] (unit normals), w[Nq]
    (area weights including a^2), t[p+1], omega[p+1]."""
    t, om = gauss_legendre(p + 1)
    theta = np.arccos(t)
    phi = np.pi * np.arange(2 * p) / p
    th, ph = np.meshgrid(theta, phi, indexing="ij")  # [p+1, 2p]; flatten -> k*2p + l
    ct = np.meshgrid(t, phi, indexing="ij")[0]       # cos(theta_k) = t_k exactly (O1: theta_k = arccos t_k)
    st = np.sqrt(1.0 - ct * ct)
    xi = np.stack([st * np.cos(ph), st * np.sin(ph), ct], axis=-1).reshape(-1, 3)
    w = (a * a * np.outer(om, np.full(2 * p, np.pi / p))).reshape(-1)
    return dict(p=p, a=a, t=t, omega=om, theta=theta, phi=phi, xi=xi, w=w,
                theta_node=th.reshape(-1), phi_node=ph.reshape(-1))


def nq(p):
    return (p + 1) * 2 * p
