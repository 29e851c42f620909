"""Mobility operator M_slip: (F, T; u_s) -> (U, Omega) (oracle; TEST INFRASTRUCTURE ONLY).

PAPER.md P:71-74 defines U = M F (vectors ordered (Fx,Fy,Fz,Tx,Ty,Tz) per particle)
and the factorisation M ~ P M^stk P^T (Fig. 1); it cites prior work for
the BIE.  Readings R1-R4, O7:

  f   = P^T(F, T) = F/(4 pi a^2) + 3/(8 pi a^3) T x xi                    (R2)
  g   = S_full[f]
  A_op q = -q/2 + D_full[q] + Pi_R[q],   Pi_R the per-sphere L2_w projector
           onto rigid motions: Pi_R[q](x) = Ubar + Obar x (x - c),
           Ubar = sum w q / (4 pi a^2),  Obar = 3/(8 pi a^4) sum w (x-c) x q
  solve A_op q = u_s - g;      (U, Omega) = -(Ubar[q], Obar[q])          (R3, R4)

GMRES here is the textbook full (unrestarted) Arnoldi + modified Gram-Schmidt +
Givens iteration from q0 = 0 to relative residual <= tol (default 1e-13).
Pins (tests/test_oracle_operator.py: test_single_sphere_mobility, test_single_janus_sphere,
test_gmres_vs_dense_solve, test_rotation_covariance, test_far_spheres_rpy): single sphere U = F/(6 pi mu a),
Omega = T/(8 pi mu a^3); single Janus sphere U = -<u_s>; GMRES vs dense LU on a
tiny scene; exact discrete covariance under z-rotation by pi/p and z-reflection;
two far spheres vs Rotne-Prager-Yamakawa.
"""
import numpy as np


def PT(disc, FT):
    """Forces/torques [Np,6] -> traction density f [N,3] (R2)."""
    FT = np.asarray(FT, dtype=np.float64).reshape(-1, 6)
    a = disc.a
    xi = disc.grid["xi"]
    F, T = FT[:, :3], FT[:, 3:]
    f = F[:, None, :] / (4.0 * np.pi * a * a) + 3.0 / (8.0 * np.pi * a ** 3) * np.cross(T[:, None, :], xi[None, :, :])
    return f.reshape(-1, 3)


def rigid_coeffs(disc, q):
    """(Ubar, Obar) per sphere [Np,6] of a density q [N,3]."""
    a = disc.a
    q = np.asarray(q).reshape(disc.np, disc.nq, 3)
    w = disc.grid["w"]
    rel = a * disc.grid["xi"]
    U = np.einsum("j,njb->nb", w, q) / (4.0 * np.pi * a * a)
    O = 3.0 / (8.0 * np.pi * a ** 4) * np.einsum("j,njb->nb", w, np.cross(rel[None, :, :], q))
    return np.concatenate([U, O], axis=1)


def rigid_field(disc, UO):
    """U + Omega x (x - c) at every node, [N,3]."""
    UO = np.asarray(UO).reshape(-1, 6)
    rel = disc.a * disc.grid["xi"]
    v = UO[:, None, :3] + np.cross(UO[:, None, 3:], rel[None, :, :])
    return v.reshape(-1, 3)


def Pi_R(disc, q):
    return rigid_field(disc, rigid_coeffs(disc, q))


def A_op(disc, q):
    q = np.asarray(q).reshape(-1, 3)
    return -0.5 * q + disc.apply_all(q=q) + Pi_R(disc, q)


def gmres(apply, rhs, tol=1e-13, maxiter=400, hist=None):
    """Textbook full GMRES (MGS Arnoldi, Givens), x0 = 0.  Returns (x, iters, relres).
    hist: optional list that receives the relative residual after every iteration."""
    b = rhs.reshape(-1)
    beta = np.linalg.norm(b)
    if beta == 0.0:
        return np.zeros_like(b), 0, 0.0
    V = [b / beta]
    H = np.zeros((maxiter + 1, maxiter))
    cs, sn = np.zeros(maxiter), np.zeros(maxiter)
    g = np.zeros(maxiter + 1)
    g[0] = beta
    k = 0
    relres = 1.0
    for k in range(maxiter):
        w = apply(V[k]).reshape(-1)
        for i in range(k + 1):
            H[i, k] = np.dot(V[i], w)
            w = w - H[i, k] * V[i]
        H[k + 1, k] = np.linalg.norm(w)
        for i in range(k):
            t = cs[i] * H[i, k] + sn[i] * H[i + 1, k]
            H[i + 1, k] = -sn[i] * H[i, k] + cs[i] * H[i + 1, k]
            H[i, k] = t
        den = np.hypot(H[k, k], H[k + 1, k])
        cs[k], sn[k] = H[k, k] / den, H[k + 1, k] / den
        H[k, k] = den
        H[k + 1, k] = 0.0
        g[k + 1] = -sn[k] * g[k]
        g[k] = cs[k] * g[k]
        relres = abs(g[k + 1]) / beta
        if hist is not None:
            hist.append(relres)
        if relres <= tol:
            break
        V.append(w / np.linalg.norm(w)) if np.linalg.norm(w) > 0 else V.append(w)
    n = k + 1
    y = np.linalg.solve(np.triu(H[:n, :n]), g[:n])
    x = sum(y[i] * V[i] for i in range(n))
    return x, n, relres


def mobility(disc, FT, slip=None, tol=1e-13, maxiter=400, return_info=False):
    """M_slip (F, T; u_s) -> (U, Omega) [Np,6] (O7)."""
    f = PT(disc, FT)
    g = disc.apply_all(f=f)
    rhs = -g if slip is None else np.asarray(slip).reshape(-1, 3) - g
    hist = []
    q, it, rr = gmres(lambda v: A_op(disc, v), rhs, tol=tol, maxiter=maxiter, hist=hist)
    UO = -rigid_coeffs(disc, q)
    if return_info:
        return UO, dict(iters=it, relres=rr, q=q.reshape(-1, 3), hist=hist)
    return UO


def janus_slip(disc, axes, B=1.0):
    """Tangential Janus slip (reading R13): on sphere m with unit axis a_m,
    u_s = -B (a_m - (xi . a_m) xi) where xi . a_m > 0, else 0."""
    axes = np.asarray(axes, dtype=np.float64).reshape(-1, 3)
    xi = disc.grid["xi"]
    out = np.zeros((disc.np, disc.nq, 3))
    for m in range(disc.np):
        c = xi @ axes[m]
        tang = axes[m][None, :] - c[:, None] * xi
        out[m] = np.where((c > 0.0)[:, None], -B * tang, 0.0)
    return out.reshape(-1, 3)
