"""Loader for the oracle's plain-C direct sum (TEST INFRASTRUCTURE ONLY).

``build()`` compiles oracle/csrc/oracle_sum.c with gcc (generic x86-64, OpenMP) to
oracle/_oracle_sum.so; __graft_entry__.build() and tests/conftest.py call it.
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "csrc", "oracle_sum.c")
_SO = os.path.join(_HERE, "_oracle_sum.so")
_lib = None


def build(force=False):
    if not force and os.path.exists(_SO) and os.path.getmtime(_SO) >= os.path.getmtime(_SRC):
        return _SO
    cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _SO, _SRC, "-lm"]
    subprocess.check_call(cmd)
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        d = ctypes.POINTER(ctypes.c_double)
        lib.oracle_direct_sum.restype = ctypes.c_long
        lib.oracle_direct_sum.argtypes = [ctypes.c_long, d, ctypes.c_long, d, d, d, d, d,
                                          ctypes.c_double, d]
        _lib = lib
    return _lib


def _ptr(a):
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def direct_sum(x, y, ny, w, f, q, mu):
    """u_i = sum_j w_j [G(x_i-y_j) f_j + K_D(x_i,y_j) q_j] (see oracle_sum.c)."""
    lib = _load()
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    ny = np.ascontiguousarray(ny, dtype=np.float64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    f = None if f is None else np.ascontiguousarray(f, dtype=np.float64)
    q = None if q is None else np.ascontiguousarray(q, dtype=np.float64)
    u = np.zeros((x.shape[0], 3))
    nz = lib.oracle_direct_sum(x.shape[0], _ptr(x), y.shape[0], _ptr(y), _ptr(ny), _ptr(w),
                               _ptr(f), _ptr(q), float(mu), _ptr(u))
    if nz:
        raise ValueError("oracle direct sum: %d coincident target/source pairs" % nz)
    return u


def far_sum(x, tsph, excl_ptr, excl, nsph, nq, y, ny, w, f, q, mu):
    """Coarse-rule far sum with per-target sphere exclusions (see oracle_sum.c)."""
    lib = _load()
    if not hasattr(lib, "_far_ready"):
        d = ctypes.POINTER(ctypes.c_double)
        lp = ctypes.POINTER(ctypes.c_long)
        lib.oracle_far_sum.restype = ctypes.c_long
        lib.oracle_far_sum.argtypes = [ctypes.c_long, d, lp, lp, lp, ctypes.c_long, ctypes.c_long,
                                       d, d, d, d, d, ctypes.c_double, d]
        lib._far_ready = True
    lp = ctypes.POINTER(ctypes.c_long)
    x = np.ascontiguousarray(x, dtype=np.float64)
    tsph = np.ascontiguousarray(tsph, dtype=np.int64)
    excl_ptr = np.ascontiguousarray(excl_ptr, dtype=np.int64)
    excl = np.ascontiguousarray(excl if len(excl) else np.zeros(1), dtype=np.int64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    ny = np.ascontiguousarray(ny, dtype=np.float64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    f = None if f is None else np.ascontiguousarray(f, dtype=np.float64)
    q = None if q is None else np.ascontiguousarray(q, dtype=np.float64)
    u = np.zeros((x.shape[0], 3))
    nz = lib.oracle_far_sum(x.shape[0], _ptr(x), tsph.ctypes.data_as(lp), excl_ptr.ctypes.data_as(lp),
                            excl.ctypes.data_as(lp), nsph, nq, _ptr(y), _ptr(ny), _ptr(w), _ptr(f),
                            _ptr(q), float(mu), _ptr(u))
    if nz:
        raise ValueError("oracle far sum: %d coincident target/source pairs" % nz)
    return u
