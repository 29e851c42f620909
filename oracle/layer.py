"""The discrete layer operator L(f, q) = S_full[f] + D_full[q] (oracle; TEST INFRASTRUCTURE ONLY).

Definition O6 (readings R5-R8), written out literally: at every node
x_i of sphere n

  u_i =   sum_{m != n, (i,m) not near} sum_{j in m} w_j [G(x_i-y_j) f_j + K_D(x_i,y_j) q_j]
        + sum_{m: (i,m) near}  sum_{s in ref(i,m)} w_s [G(x_i-y_s) f~_m(y_s) + K_D(x_i,y_s) q~_m(y_s)]
        + sum_{j in n} (S_self[i,j] f_j + D_self[i,j] q_j)

- near incidence (i, m): |x_i - c_m| - a < d_near = 4 pi a / p (R8, nearquad.py);
- ref(i, m): the refined polar sinh-graded rule of nearquad.py, f~_m the Pi_p
  interpolant of sphere m's nodal density;
- S_self / D_self: rotated-grid singular quadrature of order p_s = 2p (R5, R6).

The paper treats this operator as a black box.
Pins: tests/test_oracle_operator.py (test_direct_sum_vs_longdouble,
test_layer_far_field_and_gauss, test_layer_targets_subset_matches_all).
"""
import numpy as np

from . import native
from .grid import sphere_grid
from .nearquad import incidences, near_rule, near_tensor
from .sh import Projector
from .stokes import self_rows


def near_pairs(centers, a, dnear):
    """Unordered sphere pairs (n < m) with gap < dnear, lexicographic."""
    out = []
    np_ = centers.shape[0]
    for n in range(np_):
        for m in range(n + 1, np_):
            gap = np.linalg.norm(centers[m] - centers[n]) - 2.0 * a
            if gap < dnear:
                out.append((n, m))
    return out


class Disc:
    """One fidelity of the discretisation over a set of sphere centres."""

    def __init__(self, centers, p, a=1.0, mu=1.0, ps=None, dnear=None):
        self.centers = np.asarray(centers, dtype=np.float64).reshape(-1, 3)
        self.np = self.centers.shape[0]
        self.p, self.a, self.mu = p, a, mu
        self.ps = 2 * p if ps is None else ps
        self.dnear = 4.0 * np.pi * a / p if dnear is None else dnear
        self.rule = near_rule(p)
        self.grid = sphere_grid(p, a)
        self.nq = self.grid["xi"].shape[0]
        self.N = self.np * self.nq
        self.proj = Projector(self.grid)
        xi = self.grid["xi"]
        self.X = (self.centers[:, None, :] + a * xi[None, :, :]).reshape(-1, 3)
        self.NRM = np.tile(xi, (self.np, 1))
        self.W = np.tile(self.grid["w"], self.np)
        self.sphere_of = np.repeat(np.arange(self.np), self.nq)
        self.near = near_pairs(self.centers, a, self.dnear)
        self.inc = incidences(self.X, self.sphere_of, self.centers, a, self.dnear, self.near)
        self.inc_t = np.array([i for i, _ in self.inc], dtype=np.int64)
        self.inc_m = np.array([m for _, m in self.inc], dtype=np.int64)
        excl = [[] for _ in range(self.N)]
        for i, m in self.inc:
            excl[i].append(m)
        self.excl = excl
        self._self = {}
        self._T = {}

    # -- self blocks -------------------------------------------------------
    def self_row(self, i_local):
        if i_local not in self._self:
            self._self[i_local] = self_rows(self.grid, self.proj, i_local, self.ps, self.mu)
        return self._self[i_local]

    def self_full(self):
        S = np.zeros((self.nq, 3, self.nq, 3))
        D = np.zeros((self.nq, 3, self.nq, 3))
        for i in range(self.nq):
            S[i], D[i] = self.self_row(i)
        return S, D

    # -- near tensors ------------------------------------------------------
    def near_T(self, k):
        """T for incidence k: [2, 3, 3, nb] (see nearquad.near_tensor)."""
        if k not in self._T:
            i, m = self.inc[k]
            self._T[k] = near_tensor(self.X[i], self.centers[m], self.a, self.mu, self.p, self.rule)
        return self._T[k]

    def coefs(self, dens):
        """SH coefficients of the Pi_p interpolant per sphere: [Np, nb, 3]."""
        return np.einsum("bj,njc->nbc", self.proj.analysis, dens.reshape(self.np, self.nq, 3))

    # -- the operator ------------------------------------------------------
    def apply(self, f=None, q=None, targets=None):
        """L(f, q) at all nodes ([N,3]) or at the given global target indices."""
        if targets is None:
            targets = np.arange(self.N)
        targets = np.asarray(targets, dtype=np.int64)
        f = None if f is None else np.asarray(f, dtype=np.float64).reshape(-1, 3)
        q = None if q is None else np.asarray(q, dtype=np.float64).reshape(-1, 3)
        # far (coarse) part
        excl_ptr = np.zeros(targets.size + 1, dtype=np.int64)
        excl = []
        for k, t in enumerate(targets):
            excl.extend(self.excl[t])
            excl_ptr[k + 1] = len(excl)
        u = native.far_sum(self.X[targets], self.sphere_of[targets], excl_ptr, np.array(excl, dtype=np.int64),
                           self.np, self.nq, self.X, self.NRM, self.W, f, q, self.mu)
        # near (refined) part
        pos = {int(t): k for k, t in enumerate(targets)}
        cf = None if f is None else self.coefs(f)
        cq = None if q is None else self.coefs(q)
        for k, (i, m) in enumerate(self.inc):
            if i not in pos:
                continue
            T = self.near_T(k)
            if f is not None:
                u[pos[i]] += np.einsum("abk,kb->a", T[0], cf[m])
            if q is not None:
                u[pos[i]] += np.einsum("abk,kb->a", T[1], cq[m])
        # self part
        for k, t in enumerate(targets):
            n = int(t // self.nq)
            S_row, D_row = self.self_row(int(t - n * self.nq))
            sl = slice(n * self.nq, (n + 1) * self.nq)
            if f is not None:
                u[k] += np.einsum("ajb,jb->a", S_row, f[sl])
            if q is not None:
                u[k] += np.einsum("ajb,jb->a", D_row, q[sl])
        return u

    def apply_all(self, f=None, q=None):
        """apply() at all nodes; near and self parts vectorised (same sums)."""
        f = None if f is None else np.asarray(f, dtype=np.float64).reshape(-1, 3)
        q = None if q is None else np.asarray(q, dtype=np.float64).reshape(-1, 3)
        excl_ptr = np.zeros(self.N + 1, dtype=np.int64)
        excl_ptr[1:] = np.cumsum([len(e) for e in self.excl])
        excl = np.array([m for e in self.excl for m in e], dtype=np.int64)
        out = native.far_sum(self.X, self.sphere_of, excl_ptr, excl, self.np, self.nq, self.X,
                             self.NRM, self.W, f, q, self.mu)
        if len(self.inc):
            Tall = self.near_T_all()
            if f is not None:
                cf = self.coefs(f)
                np.add.at(out, self.inc_t, np.einsum("kabn,knb->ka", Tall[:, 0], cf[self.inc_m]))
            if q is not None:
                cq = self.coefs(q)
                np.add.at(out, self.inc_t, np.einsum("kabn,knb->ka", Tall[:, 1], cq[self.inc_m]))
        S, D = self.self_full()
        if f is not None:
            out += np.einsum("iajb,njb->nia", S, f.reshape(self.np, self.nq, 3)).reshape(-1, 3)
        if q is not None:
            out += np.einsum("iajb,njb->nia", D, q.reshape(self.np, self.nq, 3)).reshape(-1, 3)
        return out

    def near_T_all(self, workers=1):
        """All incidences' near tensors [n_inc, 2, 3, 3, nb].  workers > 1 computes the same
        per-incidence tensors (near_T) in forked worker processes writing disjoint slices of one
        shared array -- a wall-time convenience for the large fixtures, no change of arithmetic."""
        if not hasattr(self, "_Tall"):
            if not self.inc:
                self._Tall = None
            elif workers <= 1:
                self._Tall = np.stack([self.near_T(k) for k in range(len(self.inc))])
            else:
                import multiprocessing as mp
                shape = (len(self.inc),) + self.near_T(0).shape
                buf = mp.RawArray("d", int(np.prod(shape)))
                out = np.frombuffer(buf, dtype=np.float64).reshape(shape)
                bounds = np.linspace(0, shape[0], workers + 1).astype(int)

                def work(k0, k1):
                    dst = np.frombuffer(buf, dtype=np.float64).reshape(shape)
                    for k in range(k0, k1):
                        i, m = self.inc[k]
                        dst[k] = near_tensor(self.X[i], self.centers[m], self.a, self.mu, self.p, self.rule)

                ctx = mp.get_context("fork")
                procs = [ctx.Process(target=work, args=(bounds[w], bounds[w + 1])) for w in range(workers)]
                for pr in procs:
                    pr.start()
                for pr in procs:
                    pr.join()
                    if pr.exitcode != 0:
                        raise RuntimeError("near tensor worker failed")
                self._Tall = out
            self._T = {}
        return self._Tall
