"""ctypes binding of libbpqn (include/bpqn.h): argument marshalling only.

Every function has the C name without the ``bpqn_`` prefix.  Device buffers are
torch CUDA tensors (float64 / int32, contiguous); the stream is torch's current
stream unless one is given.  There is no CPU fallback: if libbpqn.so is missing
or no CUDA device is present, calls raise.
"""
import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libbpqn.so")

c_int, c_double, c_void_p, c_longlong = ctypes.c_int, ctypes.c_double, ctypes.c_void_p, ctypes.c_longlong
P = ctypes.POINTER


class DiscOpts(ctypes.Structure):
    _fields_ = [("p_s", c_int), ("d_near", c_double), ("near_n1", c_int), ("near_n2", c_int),
                ("near_nphi", c_int), ("build_single_layer", c_int), ("fmm_order", c_int)]


class GmresOpts(ctypes.Structure):
    _fields_ = [("tol", c_double), ("restart", c_int), ("max_iters", c_int), ("precond", c_int),
                ("recycle", c_int), ("relax_fmm", c_int), ("relax_delta", c_double)]


class GmresStats(ctypes.Structure):
    _fields_ = [("iters", c_int), ("restarts", c_int), ("rel_resid", c_double), ("ms", c_double),
                ("applies", c_int), ("fmm_applies", c_int)]


class SolveOpts(ctypes.Structure):
    _fields_ = [("method", c_int), ("k_max", c_int), ("eps_kkt_abs", c_double), ("eps_kkt_rel", c_double),
                ("tau", c_double), ("refresh_period", c_int), ("sub_eps_factor", c_double),
                ("sub_k_max", c_int), ("prox_tol", c_double), ("prox_jmax", c_int), ("curv_skip", c_double),
                ("gm_hi", GmresOpts), ("gm_lo", GmresOpts), ("cost_ratio", c_double), ("sub_forcing", c_double),
                ("verify_secants", c_int), ("lo_dense", c_int), ("warm_start", c_int)]


class Report(ctypes.Structure):
    _fields_ = [("iterations", c_int), ("hi_mvps", c_int), ("lo_mvps", c_int), ("gmres_iters_hi", c_int),
                ("gmres_iters_lo", c_int), ("e_mvps", c_double), ("cost_ratio", c_double),
                ("kkt_abs", c_double), ("kkt_rel", c_double), ("objective", c_double),
                ("ms_total", c_double), ("ms_hi", c_double), ("ms_lo", c_double), ("termination", c_int),
                ("secant_residual", c_double), ("lo_mvps_init", c_int), ("lo_dense_columns", c_int),
                ("lo_dense_gmres_iters", c_int), ("ms_lo_dense", c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class StepReport(ctypes.Structure):
    _fields_ = [("n_contacts", c_int), ("active_contacts", c_int), ("solve_rc", c_int),
                ("min_gap_before", c_double), ("min_gap_after", c_double), ("ms_total", c_double),
                ("lcp", Report), ("gm_nc", GmresStats), ("gm_c", GmresStats)]


ALLGATHER_FN = ctypes.CFUNCTYPE(c_int, c_void_p)

SYMBOLS = {
    "bpqn_default_disc_opts": (None, [P(DiscOpts)]),
    "bpqn_default_gmres_opts": (None, [P(GmresOpts)]),
    "bpqn_default_solve_opts": (None, [P(SolveOpts)]),
    "bpqn_geometry_init": (c_int, [P(c_void_p), c_int, c_void_p, c_double, c_double, c_int, P(DiscOpts), c_void_p]),
    "bpqn_geometry_destroy": (c_int, [c_void_p]),
    "bpqn_geometry_info": (c_int, [c_void_p, P(c_int), P(c_int), P(c_longlong), P(c_longlong)]),
    "bpqn_contacts": (c_int, [c_void_p, c_double, c_int, P(c_int), c_void_p, c_void_p, c_void_p, c_void_p]),
    "bpqn_set_contacts": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p]),
    "bpqn_layer_apply": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "bpqn_janus_slip": (c_int, [c_void_p, c_void_p, c_double, c_void_p, c_void_p]),
    "bpqn_mobility_apply": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, P(GmresOpts), P(GmresStats), c_void_p]),
    "bpqn_lcp_mvp": (c_int, [c_void_p, c_void_p, c_void_p, P(GmresOpts), P(GmresStats), c_void_p]),
    "bpqn_lcp_b": (c_int, [c_void_p, c_void_p, c_void_p, c_double, c_void_p, P(GmresOpts), P(GmresStats), c_void_p]),
    "bpqn_solve_lcp": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, P(SolveOpts), P(Report), c_void_p]),
    "bpqn_solve_lcp_dense": (c_int, [c_void_p, c_void_p, c_int, c_void_p, c_void_p, P(SolveOpts), P(Report)]),
    "bpqn_solve_lcp_dense_dev": (c_int, [c_void_p, c_void_p, c_int, c_void_p, c_void_p, P(SolveOpts), P(Report),
                                         c_void_p]),
    "bpqn_last_error": (ctypes.c_char_p, []),
    "bpqn_gmres_recycle_reset": (c_int, [c_void_p]),
    "bpqn_geometry_shard": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, ALLGATHER_FN, c_void_p]),
    "bpqn_geometry_shard_symmetric": (c_int, [c_void_p, c_void_p, c_void_p, ALLGATHER_FN, c_void_p]),
    "bpqn_nccl_unique_id": (c_int, [c_void_p]),
    "bpqn_lcp_matrix_dense": (c_int, [c_void_p, P(GmresOpts), c_void_p, P(GmresStats), c_void_p]),
    "bpqn_operator_dense": (c_int, [c_void_p, c_void_p, c_void_p]),
    "bpqn_diag_rsqrt_seed": (c_int, [c_int, c_int, P(c_double)]),
    "bpqn_geometry_shard_nccl": (c_int, [c_void_p, c_int, c_int, c_void_p, c_int]),
    "bpqn_geometry_update": (c_int, [c_void_p, c_void_p, c_void_p]),
    "bpqn_dvi_step": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_double, c_double, c_double,
                              P(SolveOpts), c_void_p, P(StepReport), c_void_p]),
    "bpqn_profile_get": (c_int, [c_void_p, P(c_double), P(c_double), P(c_double), P(c_double), P(c_longlong),
                                 P(c_longlong)]),
    "bpqn_profile_reset": (c_int, [c_void_p, c_int]),
}

_lib = None


class BpqnError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__("bpqn error %d: %s" % (code, msg))
        self.code = code


def lib():
    """Load libbpqn.so (in-tree).  Raises if it is missing -- there is no fallback."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError("libbpqn.so not built (run __graft_entry__.build() or "
                              "python paper_2604_10089_b200/build.py)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SYMBOLS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise BpqnError(rc, lib().bpqn_last_error().decode())
    return rc


def _stream(stream):
    if stream is not None:
        return ctypes.c_void_p(stream)
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t):
    if t is None:
        return None
    import torch
    assert isinstance(t, torch.Tensor) and t.is_cuda and t.is_contiguous(), "need a contiguous CUDA tensor"
    return ctypes.c_void_p(t.data_ptr())


def _hptr(a):
    import numpy as np
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(c_void_p)


def default_disc_opts():
    o = DiscOpts()
    lib().bpqn_default_disc_opts(ctypes.byref(o))
    return o


def default_gmres_opts(tol=None, restart=None, max_iters=None, precond=None, recycle=None, relax_fmm=None,
                       relax_delta=None):
    o = GmresOpts()
    lib().bpqn_default_gmres_opts(ctypes.byref(o))
    if relax_fmm is not None:
        o.relax_fmm = relax_fmm
    if relax_delta is not None:
        o.relax_delta = relax_delta
    if recycle is not None:
        o.recycle = recycle
    if precond is not None:
        o.precond = precond
    if tol is not None:
        o.tol = tol
    if restart is not None:
        o.restart = restart
    if max_iters is not None:
        o.max_iters = max_iters
    return o


def default_solve_opts(**kw):
    o = SolveOpts()
    lib().bpqn_default_solve_opts(ctypes.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


class Geometry:
    """Owning wrapper of a bpqn_geom_t handle."""

    def __init__(self, centers, p, radius=1.0, mu=1.0, opts=None, stream=None):
        import numpy as np
        c, cp = _hptr(np.asarray(centers, dtype=np.float64).reshape(-1, 3))
        h = c_void_p()
        self.np = c.shape[0]
        self.p = p
        _check(lib().bpqn_geometry_init(ctypes.byref(h), self.np, cp, radius, mu, p,
                                        ctypes.byref(opts) if opts is not None else None, _stream(stream)))
        self.h = h
        n, nq, ninc, nbytes = c_int(), c_int(), c_longlong(), c_longlong()
        _check(lib().bpqn_geometry_info(h, ctypes.byref(n), ctypes.byref(nq), ctypes.byref(ninc), ctypes.byref(nbytes)))
        self.N, self.nq, self.n_incidences, self.device_bytes = n.value, nq.value, ninc.value, nbytes.value
        self.nc = 0

    def close(self):
        if getattr(self, "h", None):
            lib().bpqn_geometry_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def geometry_init(centers, p, radius=1.0, mu=1.0, opts=None, stream=None):
    return Geometry(centers, p, radius, mu, opts, stream)


def contacts(g, gap_threshold, max_contacts=None, stream=None):
    """Returns (pairs int32 [Nc,2], normals [Nc,3], gaps [Nc]) as CUDA tensors."""
    import torch
    cap = max_contacts if max_contacts is not None else g.np * (g.np - 1) // 2
    cap = max(cap, 1)
    pairs = torch.empty((cap, 2), dtype=torch.int32, device="cuda")
    nrm = torch.empty((cap, 3), dtype=torch.float64, device="cuda")
    gaps = torch.empty((cap,), dtype=torch.float64, device="cuda")
    n = c_int()
    _check(lib().bpqn_contacts(g.h, gap_threshold, cap, ctypes.byref(n), _ptr(pairs), _ptr(nrm), _ptr(gaps),
                               _stream(stream)))
    g.nc = n.value
    return pairs[: n.value], nrm[: n.value], gaps[: n.value]


def set_contacts(g, pairs, normals, gaps, stream=None):
    _check(lib().bpqn_set_contacts(g.h, int(pairs.shape[0]), _ptr(pairs.contiguous()), _ptr(normals.contiguous()),
                                   _ptr(gaps.contiguous()), _stream(stream)))
    g.nc = int(pairs.shape[0])


def layer_apply(g, f=None, q=None, out=None, stream=None):
    import torch
    if out is None:
        out = torch.empty((g.N, 3), dtype=torch.float64, device="cuda")
    _check(lib().bpqn_layer_apply(g.h, _ptr(f), _ptr(q), _ptr(out), _stream(stream)))
    return out


def janus_slip(g, axes, B=1.0, out=None, stream=None):
    import torch
    if out is None:
        out = torch.empty((g.N, 3), dtype=torch.float64, device="cuda")
    a, ap = _hptr(axes)
    _check(lib().bpqn_janus_slip(g.h, ap, B, _ptr(out), _stream(stream)))
    return out


def mobility_apply(g, ft, slip=None, out=None, gmres=None, stream=None):
    import torch
    if out is None:
        out = torch.empty((g.np, 6), dtype=torch.float64, device="cuda")
    st = GmresStats()
    _check(lib().bpqn_mobility_apply(g.h, _ptr(ft), _ptr(slip), _ptr(out),
                                     ctypes.byref(gmres) if gmres is not None else None, ctypes.byref(st),
                                     _stream(stream)))
    return out, st


def lcp_mvp(g, lam, out=None, gmres=None, stream=None):
    import torch
    if out is None:
        out = torch.empty((g.nc,), dtype=torch.float64, device="cuda")
    st = GmresStats()
    _check(lib().bpqn_lcp_mvp(g.h, _ptr(lam), _ptr(out), ctypes.byref(gmres) if gmres is not None else None,
                              ctypes.byref(st), _stream(stream)))
    return out, st


def lcp_b(g, fnc, slip=None, dt=1.0, out=None, gmres=None, stream=None):
    import torch
    if out is None:
        out = torch.empty((g.nc,), dtype=torch.float64, device="cuda")
    st = GmresStats()
    _check(lib().bpqn_lcp_b(g.h, _ptr(fnc), _ptr(slip), dt, _ptr(out),
                            ctypes.byref(gmres) if gmres is not None else None, ctypes.byref(st), _stream(stream)))
    return out, st


def solve_lcp(hi, lo, b, lam, opts=None, stream=None):
    """lam (CUDA float64 [Nc]) is the initial guess on input and the solution on output."""
    rep = Report()
    rc = lib().bpqn_solve_lcp(hi.h, lo.h if lo is not None else None, _ptr(b), _ptr(lam),
                              ctypes.byref(opts) if opts is not None else None, ctypes.byref(rep), _stream(stream))
    if rc not in (0, 4, 5):
        _check(rc)
    return lam, rep, rc


def solve_lcp_dense(A, b, x0=None, Ahat=None, opts=None):
    import numpy as np
    A, Ap = _hptr(A)
    n = A.shape[0]
    b, bp = _hptr(b)
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=np.float64)
    x, xp = _hptr(x)
    if Ahat is not None:
        Ah, Ahp = _hptr(Ahat)
    else:
        Ahp = None
    rep = Report()
    rc = lib().bpqn_solve_lcp_dense(Ap, Ahp, n, bp, xp, ctypes.byref(opts) if opts is not None else None,
                                    ctypes.byref(rep))
    if rc not in (0, 4, 5):
        _check(rc)
    return x, rep, rc


def solve_lcp_dense_dev(A, b, x, Ahat=None, opts=None, stream=None):
    """Dense LCP solve with CUDA tensors (x: initial guess in, solution out)."""
    rep = Report()
    rc = lib().bpqn_solve_lcp_dense_dev(_ptr(A), _ptr(Ahat), int(b.shape[0]), _ptr(b), _ptr(x),
                                        ctypes.byref(opts) if opts is not None else None, ctypes.byref(rep),
                                        _stream(stream))
    if rc not in (0, 4, 5):
        _check(rc)
    return x, rep, rc


def geometry_update(g, centers, stream=None):
    """Move the handle to new centres (same spheres, p); clears its contact set."""
    import numpy as np
    c, cp = _hptr(np.asarray(centers, dtype=np.float64).reshape(-1, 3))
    _check(lib().bpqn_geometry_update(g.h, cp, _stream(stream)))
    g.nc = 0


def dvi_step(hi, lo, centers, axes, fnc, slip_B=1.0, dt=1.0, delta=0.1, opts=None, stream=None):
    """One DVI time step (bpqn_dvi_step).  centers / axes (numpy [Np,3]) are updated in
    place; returns ((U, Omega) [Np,6], StepReport, rc)."""
    import numpy as np
    assert centers.dtype == np.float64 and centers.flags.c_contiguous
    assert axes.dtype == np.float64 and axes.flags.c_contiguous
    f, fp = _hptr(np.asarray(fnc, dtype=np.float64).reshape(-1, 3))
    uo = np.zeros((hi.np, 6))
    rep = StepReport()
    rc = lib().bpqn_dvi_step(hi.h, lo.h if lo is not None else None, centers.ctypes.data_as(c_void_p),
                             axes.ctypes.data_as(c_void_p), fp, slip_B, dt, delta,
                             ctypes.byref(opts) if opts is not None else None, uo.ctypes.data_as(c_void_p),
                             ctypes.byref(rep), _stream(stream))
    if rc not in (0, 4, 5):
        _check(rc)
    hi.nc = 0
    if lo is not None:
        lo.nc = 0
    return uo, rep, rc


def _torch_allgather(send, recv):
    """all-gather of equal-size device buffers with torch.distributed (NCCL directly; other
    backends, e.g. gloo in tests, through host copies)."""
    import torch
    import torch.distributed as dist
    if dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(recv, send)
    else:
        parts = [torch.empty(send.numel(), dtype=send.dtype) for _ in range(dist.get_world_size())]
        dist.all_gather(parts, send.cpu())
        recv.copy_(torch.cat(parts).to(recv.device))
    torch.cuda.current_stream().synchronize()


def _torch_reduce_scatter(send, recv):
    """reduce-scatter (sum) of [world][rows] device buffers with torch.distributed (NCCL directly;
    other backends, e.g. gloo in tests, as an all-reduce of host copies)."""
    import torch
    import torch.distributed as dist
    if dist.get_backend() == "nccl":
        dist.reduce_scatter_tensor(recv, send)
    else:
        h = send.cpu()
        dist.all_reduce(h)
        r, n = dist.get_rank(), recv.numel()
        recv.copy_(h[r * n:(r + 1) * n].to(recv.device))
    torch.cuda.current_stream().synchronize()


def _callback(fn, a, b):
    def cb(_user):
        try:
            fn(a, b)
            return 0
        except Exception:  # reported as BPQN_ERR_CUDA by the library
            import traceback
            traceback.print_exc()
            return 1
    return ALLGATHER_FN(cb)


def geometry_shard(g, rank, world, allgather=None, symmetric=False, reduce_scatter=None):
    """Shard the layer operator's target side over `world` ranks (bpqn_geometry_shard);
    `allgather(send, recv)` performs the collective on the two CUDA tensors (default:
    torch.distributed).  symmetric=True also runs K1 as the symmetric kernel split over the
    ranks (bpqn_geometry_shard_symmetric) with `reduce_scatter(send, recv)` (default:
    torch.distributed).  world = 1 restores the single-GPU operator."""
    import torch
    if world == 1:
        _check(lib().bpqn_geometry_shard(g.h, 0, 1, None, None, ALLGATHER_FN(0), None))
        g._shard = None
        return
    rows = -(-g.np // world) * g.nq
    send = torch.zeros(3 * rows, dtype=torch.float64, device="cuda")
    recv = torch.zeros(world * 3 * rows, dtype=torch.float64, device="cuda")
    fn = allgather or _torch_allgather

    def cb(_user):
        try:
            fn(send, recv)
            return 0
        except Exception:  # reported as BPQN_ERR_CUDA by the library
            import traceback
            traceback.print_exc()
            return 1

    cfun = ALLGATHER_FN(cb)
    g._shard = (send, recv, cfun)  # keep alive as long as the sharding
    _check(lib().bpqn_geometry_shard(g.h, rank, world, _ptr(send), _ptr(recv), cfun, None))
    if symmetric:
        rs_send = torch.zeros(world * 3 * rows, dtype=torch.float64, device="cuda")
        rs_recv = torch.zeros(3 * rows, dtype=torch.float64, device="cuda")
        rfun = _callback(reduce_scatter or _torch_reduce_scatter, rs_send, rs_recv)
        g._shard = g._shard + (rs_send, rs_recv, rfun)
        _check(lib().bpqn_geometry_shard_symmetric(g.h, _ptr(rs_send), _ptr(rs_recv), rfun, None))


def diag_rsqrt_seed(exp_lo, exp_hi):
    """max |1 - rr y^2| of the MUFU.RSQ64H seed over every high-word pattern with exponents in range."""
    v = c_double()
    _check(lib().bpqn_diag_rsqrt_seed(exp_lo, exp_hi, ctypes.byref(v)))
    return v.value


def lcp_matrix_dense(g, gmres=None, stream=None):
    """A = D^T M D of the handle's contact set as a numpy [Nc, Nc] array (bpqn_lcp_matrix_dense)."""
    import numpy as np
    A = np.zeros((g.nc, g.nc))
    st = GmresStats()
    _check(lib().bpqn_lcp_matrix_dense(g.h, ctypes.byref(gmres) if gmres is not None else None,
                                       A.ctypes.data_as(c_void_p), ctypes.byref(st), _stream(stream)))
    return A, st


def operator_dense(g, out=None, stream=None):
    """The completed double-layer operator as a dense CUDA tensor [3N, 3N] (bpqn_operator_dense)."""
    import torch
    n = 3 * g.N
    if out is None:
        out = torch.empty((n, n), dtype=torch.float64, device="cuda")
    _check(lib().bpqn_operator_dense(g.h, _ptr(out), _stream(stream)))
    return out


def nccl_unique_id():
    """128 bytes for bpqn_geometry_shard_nccl (call on one rank, distribute to all)."""
    buf = ctypes.create_string_buffer(128)
    _check(lib().bpqn_nccl_unique_id(buf))
    return buf.raw


def geometry_shard_nccl(g, rank, world, uid, symmetric=True):
    """Shard the operator over `world` ranks with the library's own NCCL communicator
    (bpqn_geometry_shard_nccl; collective: every rank calls it with the same 128-byte uid)."""
    assert isinstance(uid, (bytes, bytearray)) and len(uid) == 128
    buf = ctypes.create_string_buffer(bytes(uid), 128)
    _check(lib().bpqn_geometry_shard_nccl(g.h, rank, world, buf, 1 if symmetric else 0))
    g._shard = None


def gmres_recycle_reset(g):
    _check(lib().bpqn_gmres_recycle_reset(g.h))


def profile_reset(g, events=True):
    _check(lib().bpqn_profile_reset(g.h, 1 if events else 0))


def profile_get(g):
    a, b, c, gf = c_double(), c_double(), c_double(), c_double()
    n1, n2 = c_longlong(), c_longlong()
    _check(lib().bpqn_profile_get(g.h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c), ctypes.byref(gf),
                                  ctypes.byref(n1), ctypes.byref(n2)))
    return dict(ms_allpairs=a.value, ms_near=b.value, ms_self=c.value, allpairs_gflop=gf.value,
                allpairs_launches=n1.value, kernel_launches=n2.value)
