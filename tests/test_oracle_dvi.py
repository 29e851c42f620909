"""Pins of the oracle DVI step (oracle/dvi.py)."""
import numpy as np

from oracle import dvi, mobility as mob
from oracle.layer import Disc


def test_no_contacts_is_free_mobility_step():
    """Far-apart spheres: no LCP, c^{i+1} = c^i + dt U_nc (eq. dvi with x = 0)."""
    C = np.array([[0.0, 0.0, 0.0], [4.0, 0.3, 0.0]])
    axes = np.array([[0.0, 0.0, 1.0], [1.0, 0.0, 0.0]])
    F = np.array([[0.5, 0.0, 0.0], [-0.5, 0.1, 0.0]])
    nc, na, U, lam, pairs = dvi.dvi_step(C, axes, F, p=5, dt=0.3)
    assert len(pairs) == 0
    d = Disc(C, 5)
    FT = np.zeros((2, 6))
    FT[:, :3] = F
    Uref = mob.mobility(d, FT, mob.janus_slip(d, axes, 1.0))
    np.testing.assert_allclose(nc, C + 0.3 * Uref[:, :3], atol=1e-13)


def test_pushed_pair_stops_at_contact():
    """Two spheres driven together (gap 0.02, no slip): the LCP makes the linearised gap
    Phi + dt n.(U_j - U_i) exactly 0 with lambda > 0 (complementarity),
    whereas the free step would overlap."""
    C = np.array([[0.0, 0.0, 0.0], [2.02, 0.0, 0.0]])
    axes = np.array([[0.0, 0.0, 1.0], [0.0, 0.0, 1.0]])
    dt = 1.0
    # weak push: the lubricated approach keeps the linearised gap positive, lambda = 0
    F = np.array([[1.0, 0.0, 0.0], [-1.0, 0.0, 0.0]])
    nc, na, U, lam, pairs = dvi.dvi_step(C, axes, F, p=6, dt=dt, slip_B=0.0)
    assert len(pairs) == 1 and lam[0] == 0.0 and 0.02 + dt * (U[1, 0] - U[0, 0]) > 0
    # 10x the push would close the gap (free approach is linear in F): the contact activates
    F = 10 * F
    nc, na, U, lam, pairs = dvi.dvi_step(C, axes, F, p=6, dt=dt, slip_B=0.0)
    assert lam[0] > 0
    assert abs(0.02 + dt * (U[1, 0] - U[0, 0])) < 1e-12
    assert np.allclose(U[:, 1:], 0.0, atol=1e-12)   # axial symmetry of the pair


def test_free_janus_sphere_swims_along_axis():
    """A single Janus sphere with F = 0 moves along its axis with U = -<u_s> (App. A.5),
    -> (B/3) a as p grows; Omega = 0 keeps the axis fixed."""
    a_ax = np.array([[0.36, 0.48, 0.8]])
    nc, na, U, lam, pairs = dvi.dvi_step(np.zeros((1, 3)), a_ax, np.zeros((1, 3)), p=12, dt=1.0)
    np.testing.assert_allclose(U[0, :3], a_ax[0] / 3.0, atol=1e-6)      # U = (B/3) a
    assert np.linalg.norm(U[0, 3:]) < 1e-2                               # Omega -> 0 with p
    assert abs(np.linalg.norm(na) - 1.0) < 1e-14
    np.testing.assert_allclose(na[0], a_ax[0] + np.cross(U[0, 3:], a_ax[0]), atol=1e-4)
