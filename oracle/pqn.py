"""Mono-PQN, Bi-PQN and their pieces, written out literally (oracle; TEST INFRASTRUCTURE ONLY).

Follows PAPER.md in the paper's order and notation, with the readings of SURVEY
8(c) / DESIGN.md where the text is garbled or silent:

* Alg. 1 Mono-PQN, forward step x~ = x - tau H (A x + b) (R11),
  H0 = I, tau = 1 (R19), full-memory BFGS in U/V form B = I + UU^T - VV^T (R16,
  App. D.1), curvature skip y^T s <= 1e-12 |s||y| (R16);
* the weighted prox via Prop. 1 solved by Alg. 4 semi-smooth Newton
   on the residual with the "+[alpha; alpha~]" term restored (R15):
      L(a, a~) = [a + U^T (y - z); a~ + V^T (x~ - z)],
      y = x~ + C^{-1} V a~, z = (y - D^{-1} U a)_+, C = D + UU^T,
  Jacobian = the block matrix of P:709-712 (+I);  C^{-1} by a DENSE solve (plain);
* Alg. 2 optimal over-relaxation with the tie rules of R17;
* the gradient cache A x_{k+1} = A x_k + eta A p_k (Remark P:390-392), refreshed
  every 20 iterations (R18);
* KKT errors eq. (kkt-error) P:531-533 in the Euclidean norm (R12);
* BB-PGD: projected gradient with the spectral step eq.
  (spectralStepSize); first step tau = 1 and a non-positive BB denominator reuses
  the previous tau (R31); one MVP per iteration
  on the new iterate (A x_{k+1} directly, no cache drift);
* Alg. 3 Bi-PQN with the subproblem eq. (pqnSubproblem) P:468-470,
  secant re-use P:475-487, cached low-fidelity secant A^ s = eta(A^ x^ - A^ x)
  (App. D.2), sub-solver settings R22.  The re-used secants follow the
  paper's stated requirement B^(k+1) S = Y rather than its printed
  display (P:486 / Alg. 3, "Y^ - (uu^T - vv^T) S^"): with y' = B^(k) s' the
  pair for B^(k+1) = B^(k) + uu^T - vv^T is Y = Y^ + (uu^T - vv^T) S^ (reading R34,
  DESIGN.md; pinned by SPEC S:229's dense identity in tests/test_oracle_pqn.py).

Pins: tests/test_oracle_pqn.py (SPEC.md unit vectors S:62-64, S:147, S:197-199,
S:215-217; prox vs a dense QP on 500 random
cases; eta* vs a grid; CG equivalence; brute-force LCP agreement).
"""
import numpy as np

TERM_KKT_ABS, TERM_KKT_REL, TERM_MAX_ITER, TERM_STALLED = 0, 1, 2, 3


def kkt_errors(x, g, prev_abs=None):
    """eq. (kkt-error): abs = ||min(x, Ax+b)||_2, rel = |abs - prev|/max(abs, prev)."""
    e = float(np.linalg.norm(np.minimum(x, g)))
    if prev_abs is None:
        return e, np.inf
    den = max(e, prev_abs)
    return e, (abs(e - prev_abs) / den if den > 0 else 0.0)


class BFGS:
    """Full-memory BFGS model B = I + sum u u^T - sum v v^T, inverse H by the
    classical two-loop recursion on the accepted (s, y) pairs with H0 = I."""

    def __init__(self, n):
        self.n = n
        self.U, self.V, self.S, self.Y = [], [], [], []

    def Umat(self):
        return np.stack(self.U, axis=1) if self.U else np.zeros((self.n, 0))

    def Vmat(self):
        return np.stack(self.V, axis=1) if self.V else np.zeros((self.n, 0))

    def B(self, x):
        out = np.array(x, dtype=np.float64, copy=True)
        for u in self.U:
            out += u * np.dot(u, x)
        for v in self.V:
            out -= v * np.dot(v, x)
        return out

    def H(self, g):
        q = np.array(g, dtype=np.float64, copy=True)
        alphas = []
        for s, y in zip(reversed(self.S), reversed(self.Y)):
            rho = 1.0 / np.dot(y, s)
            a = rho * np.dot(s, q)
            alphas.append(a)
            q -= a * y
        r = q  # H0 = I
        for (s, y), a in zip(zip(self.S, self.Y), reversed(alphas)):
            rho = 1.0 / np.dot(y, s)
            beta = rho * np.dot(y, r)
            r += s * (a - beta)
        return r

    def update(self, s, y, Bs=None, curv=1e-12):
        ys = float(np.dot(y, s))
        if not np.isfinite(ys):
            raise FloatingPointError("NaN in BFGS update")
        if ys <= curv * np.linalg.norm(s) * np.linalg.norm(y):
            return False
        if Bs is None:
            Bs = self.B(s)
        sBs = float(np.dot(s, Bs))
        if sBs <= 0.0:
            return False
        self.U.append(y / np.sqrt(ys))
        self.V.append(Bs / np.sqrt(sBs))
        self.S.append(np.array(s, copy=True))
        self.Y.append(np.array(y, copy=True))
        return True


def prox_residual(Dg, U, V, xt, a, at):
    """L(a, a~) of Prop. 1 with the R15 correction; returns (L, z, Lambda)."""
    C = np.diag(Dg) + U @ U.T
    CinvV = np.linalg.solve(C, V) if V.shape[1] else np.zeros((xt.size, 0))
    DinvU = U / Dg[:, None]
    y = xt + CinvV @ at
    arg = y - DinvU @ a
    z = np.maximum(arg, 0.0)
    lam = (z > 0.0).astype(np.float64)
    L = np.concatenate([a + U.T @ (y - z), at + V.T @ (xt - z)])
    return L, z, lam


def prox_jacobian(Dg, U, V, lam):
    """J_L of P:709-712 (+ I)."""
    C = np.diag(Dg) + U @ U.T
    CinvV = np.linalg.solve(C, V) if V.shape[1] else np.zeros((Dg.size, 0))
    DinvU = U / Dg[:, None]
    LD = lam[:, None] * DinvU
    LC = lam[:, None] * CinvV
    top = np.concatenate([U.T @ LD, U.T @ (CinvV - LC)], axis=1)
    bot = np.concatenate([V.T @ LD, -V.T @ LC], axis=1)
    J = np.concatenate([top, bot], axis=0)
    return J + np.eye(J.shape[0])


def weighted_prox(Dg, U, V, xt, tol=None, jmax=100):
    """prox^B_{x>=0}(x~), B = diag(Dg) + UU^T - VV^T, by Alg. 4 (semi-smooth Newton),
    damped by step halving on ||L||_inf with a Tikhonov fallback.
    Returns (x_hat, iters, final ||L||_inf)."""
    xt = np.asarray(xt, dtype=np.float64)
    Dg = np.asarray(Dg, dtype=np.float64)
    ru, rv = U.shape[1], V.shape[1]
    if ru + rv == 0:
        return np.maximum(xt, 0.0), 0, 0.0
    if tol is None:
        tol = 1e-12 * max(1.0, np.abs(xt).max())
    a, at = np.zeros(ru), np.zeros(rv)
    L, z, lam = prox_residual(Dg, U, V, xt, a, at)
    nrm = np.abs(L).max()
    j = 0
    for j in range(jmax):
        if nrm <= tol:
            break
        J = prox_jacobian(Dg, U, V, lam)
        try:
            d = -np.linalg.solve(J, L)
        except np.linalg.LinAlgError:
            d = -np.linalg.solve(J + 1e-10 * np.abs(J).sum(axis=1).max() * np.eye(J.shape[0]), L)
        t = 1.0
        accepted = False
        for _ in range(30):
            a2, at2 = a + t * d[:ru], at + t * d[ru:]
            L2, z2, lam2 = prox_residual(Dg, U, V, xt, a2, at2)
            n2 = np.abs(L2).max()
            if n2 < nrm or n2 <= tol:
                accepted = True
                break
            t *= 0.5
        if not accepted:
            break
        step = t * np.abs(d).max()
        a, at, L, z, lam, nrm = a2, at2, L2, z2, lam2, n2
        if step < tol:
            break
    return z, j, nrm


def optimal_eta(x, p, g, Ap):
    """Alg. 2: eta* = min(eta', min_{p_l<0} -x_l/p_l), eta' = -p^T g / p^T A p.
    Returns (eta, binding_mask or None)."""
    pAp = float(np.dot(p, Ap))
    pg = float(np.dot(p, g))
    eta_u = -pg / pAp if pAp > 0.0 else np.inf
    neg = p < 0.0
    if neg.any():
        cand = -x[neg] / p[neg]
        eta_h = float(cand.min())
    else:
        eta_h = np.inf
    if eta_h < eta_u:
        bind = np.zeros(x.size, dtype=bool)
        idx = np.nonzero(neg)[0]
        bind[idx[cand == eta_h]] = True
        return eta_h, bind
    return eta_u, None


class Report(dict):
    pass


def mono_pqn(mvp, b, x0, eps_abs=1e-10, eps_rel=0.0, k_max=200, tau=1.0, refresh=20,
             g0=None, aux0=None, seed_pairs=(), prox_tol=None, prox_jmax=100, curv=1e-12):
    """Alg. 1.  ``mvp(v) -> (A v, aux(v))`` where aux is any linear side quantity
    to track alongside the cached gradient (Bi-PQN tracks the A^-part).  If g0 is
    given the initial MVP is skipped (subproblem warm start, no MVP).
    Returns (x, g, aux_x, pairs, report)."""
    n = b.size
    x = np.array(x0, dtype=np.float64, copy=True)
    mvps = 0
    if g0 is None:
        Ax, aux_x = mvp(x)
        mvps += 1
        g = Ax + b
    else:
        g = np.array(g0, dtype=np.float64, copy=True)
        aux_x = None if aux0 is None else np.array(aux0, dtype=np.float64, copy=True)
    qn = BFGS(n)
    for (s, y) in seed_pairs:
        qn.update(s, y, curv=curv)
    trace = []
    xs = [x.copy()]
    prev = None
    it = 0
    term = TERM_MAX_ITER
    reset_done = False
    for k in range(k_max):
        e_abs, e_rel = kkt_errors(x, g, prev)
        prev = e_abs
        trace.append(e_abs)
        if e_abs <= eps_abs:
            term = TERM_KKT_ABS
            break
        if eps_rel > 0 and e_rel <= eps_rel:
            term = TERM_KKT_REL
            break
        xt = x - tau * qn.H(g)
        xh, _, _ = weighted_prox(np.ones(n), qn.Umat(), qn.Vmat(), xt, prox_tol, prox_jmax)
        p = xh - x
        Ap, aux_p = mvp(p)
        mvps += 1
        eta, bind = optimal_eta(x, p, g, Ap)
        if not (eta > 0.0 and np.isfinite(eta)) or np.dot(p, g) >= 0.0:
            if reset_done:
                term = TERM_STALLED
                break
            qn = BFGS(n)
            reset_done = True
            continue
        reset_done = False
        x = x + eta * p
        if bind is not None:
            x[bind] = 0.0
        g = g + eta * Ap
        xs.append(x.copy())
        if aux_x is not None and aux_p is not None:
            aux_x = aux_x + eta * aux_p
        it += 1
        s, y = eta * p, eta * Ap
        qn.update(s, y, curv=curv)
        if refresh and it % refresh == 0:
            Ax, aux_x = mvp(x)
            mvps += 1
            g = Ax + b
    else:
        e_abs, _ = kkt_errors(x, g, prev)
        trace.append(e_abs)
    pairs = list(zip(qn.S, qn.Y))
    rep = Report(iterations=it, mvps=mvps, termination=term, kkt_abs=trace[-1],
                 kkt_trace=trace, x_trace=xs, objective=float(0.5 * np.dot(x, g - b) + np.dot(x, b)))
    return x, g, aux_x, pairs, rep


def bb_step(s, As, tau_prev):
    """eq. (spectralStepSize): tau_bb = ||s||^2 / s^T A s; a non-positive denominator
    reuses the previous tau."""
    den = float(np.dot(s, As))
    return float(np.dot(s, s)) / den if den > 0.0 else tau_prev


def bb_pgd(mvp, b, x0, eps_abs=1e-10, eps_rel=0.0, k_max=500):
    """BB-PGD: x_{k+1} = (x_k - tau_k (A x_k + b))_+ with tau_0 = 1, tau_k = tau_bb
    of the last step.  ``mvp(v) -> A v``.  Returns (x, g, report)."""
    x = np.maximum(np.array(x0, dtype=np.float64), 0.0)
    g = mvp(x) + b
    mvps = 1
    tau = 1.0
    prev = None
    trace = []
    it = 0
    term = TERM_MAX_ITER
    for k in range(k_max):
        e_abs, e_rel = kkt_errors(x, g, prev)
        prev = e_abs
        trace.append(e_abs)
        if e_abs <= eps_abs:
            term = TERM_KKT_ABS
            break
        if eps_rel > 0 and e_rel <= eps_rel:
            term = TERM_KKT_REL
            break
        x_new = np.maximum(x - tau * g, 0.0)
        g_new = mvp(x_new) + b
        mvps += 1
        s, As = x_new - x, g_new - g
        tau = bb_step(s, As, tau)
        x, g = x_new, g_new
        it += 1
    else:
        trace.append(kkt_errors(x, g, prev)[0])
    rep = Report(iterations=it, mvps=mvps, termination=term, kkt_abs=trace[-1], kkt_trace=trace)
    return x, g, rep


def transform_secants(S_hat, Y_hat, u, v):
    """Secant re-use across Bi-PQN subproblems (reading R34): pairs with
    B^(k) S^ = Y^ become pairs of B^(k+1) = B^(k) + u u^T - v v^T, i.e.
    S = S^,  Y = Y^ + (u u^T - v v^T) S^."""
    return [yp + u * np.dot(u, sp) - v * np.dot(v, sp) for sp, yp in zip(S_hat, Y_hat)]


def bi_pqn(mvp_hi, mvp_lo, b, x_init, eps_abs=1e-10, eps_rel=0.0, k_max=100,
           sub_eps_factor=1e-2, sub_k_max=50, refresh=20, curv=1e-12, prox_tol=None,
           verify_secants=False):
    """Alg. 3.  mvp_hi(v) -> A v, mvp_lo(v) -> A^ v.  Returns (x, report).
    verify_secants: before every subproblem, record max_j |B^(k) s_j - y_j|_inf /
    max(1, |y_j|_inf) over the seeded pairs (extra lo MVPs, not counted; tests only)."""
    n = b.size
    cnt = dict(hi=0, lo=0)

    def lo_op(v):
        cnt["lo"] += 1
        r = mvp_lo(v)
        return r, r

    # low-fidelity initialisation x0 = Mono-PQN(A^, b, x^{-1})
    x, g_lo, Ahat_x, pairs, rep0 = mono_pqn(lo_op, b, x_init, eps_abs=eps_abs, eps_rel=eps_rel,
                                            k_max=k_max, refresh=refresh, curv=curv,
                                            prox_tol=prox_tol)
    S_low = [s for s, _ in pairs]
    Y_low = [y for _, y in pairs]
    cnt["hi"] += 1
    g = mvp_hi(x) + b
    U, V = [], []

    def Bhi(v, Ahat_v):
        out = np.array(Ahat_v, copy=True)
        for u in U:
            out += u * np.dot(u, v)
        for vv in V:
            out -= vv * np.dot(vv, v)
        return out

    trace, prev, it, term = [], None, 0, TERM_MAX_ITER
    sub_iters = []
    secant_res = []
    for k in range(k_max):
        e_abs, e_rel = kkt_errors(x, g, prev)
        prev = e_abs
        trace.append(e_abs)
        if e_abs <= eps_abs:
            term = TERM_KKT_ABS
            break
        if eps_rel > 0 and e_rel <= eps_rel:
            term = TERM_KKT_REL
            break
        c = g - Bhi(x, Ahat_x)
        if verify_secants:
            secant_res.append(max([0.0] + [float(np.abs(Bhi(sp, mvp_lo(sp)) - yp).max() /
                                                 max(1.0, np.abs(yp).max()))
                                           for sp, yp in zip(S_low, Y_low)]))

        def sub_op(v):
            cnt["lo"] += 1
            Av = mvp_lo(v)
            return Bhi(v, Av), Av

        xh, _, Ahat_xh, sub_pairs, rsub = mono_pqn(
            sub_op, c, x, eps_abs=sub_eps_factor * eps_abs, eps_rel=0.0, k_max=sub_k_max,
            refresh=refresh, g0=g, aux0=Ahat_x, seed_pairs=list(zip(S_low, Y_low)), curv=curv,
            prox_tol=prox_tol)
        sub_iters.append(rsub["iterations"])
        p = xh - x
        cnt["hi"] += 1
        Ap = mvp_hi(p)
        eta, bind = optimal_eta(x, p, g, Ap)
        if not (eta > 0.0 and np.isfinite(eta)):
            term = TERM_STALLED
            break
        x = x + eta * p
        if bind is not None:
            x[bind] = 0.0
        g = g + eta * Ap
        it += 1
        s, y = eta * p, eta * Ap
        Ahat_s = eta * (Ahat_xh - Ahat_x)
        Bs = Bhi(s, Ahat_s)
        ys, sBs = float(np.dot(y, s)), float(np.dot(s, Bs))
        S_low = [sp for sp, _ in sub_pairs]
        Y_low = [yp for _, yp in sub_pairs]
        if ys > curv * np.linalg.norm(s) * np.linalg.norm(y) and sBs > 0.0:
            u = y / np.sqrt(ys)
            v = Bs / np.sqrt(sBs)
            U.append(u)
            V.append(v)
            Y_low = transform_secants(S_low, Y_low, u, v)
        Ahat_x = Ahat_x + Ahat_s
        if refresh and it % refresh == 0:
            cnt["hi"] += 1
            g = mvp_hi(x) + b
    else:
        e_abs, _ = kkt_errors(x, g, prev)
        trace.append(e_abs)
    rep = Report(iterations=it, hi_mvps=cnt["hi"], lo_mvps=cnt["lo"], termination=term,
                 kkt_abs=trace[-1], kkt_trace=trace, init_iterations=rep0["iterations"],
                 sub_iterations=sub_iters, secant_residuals=secant_res)
    return x, rep
