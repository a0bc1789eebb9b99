"""TEST INFRASTRUCTURE ONLY -- ctypes front-end of the CPU parity oracle.

Wraps oracle/liboracle.so (a C restatement of the reference hot path,
/root/reference/pkg/src/streamforge/_kernels.py and core.py; see the file:line
citations in sfb_oracle.c).  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference arm may import this module.  The product
package never does.

The signatures mirror the reference `_kernels` seam:
arrays are numpy, stream states are the reference's int64 (n, 6) layout and are
mutated in place.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None

_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)
_f32p = ctypes.POINTER(ctypes.c_float)


def build():
    """Compile the oracle (gcc, -ffp-contract=off, OpenMP)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        L = ctypes.CDLL(_SO)
        L.orc_step.argtypes = [_i64p]
        L.orc_step.restype = ctypes.c_int64
        L.orc_fill_real.argtypes = [_i64p, _f64p] + [ctypes.c_int64] * 5 + [
            ctypes.c_int, ctypes.c_double, ctypes.c_int]
        L.orc_fill_integer.argtypes = [_i64p, _i64p] + [ctypes.c_int64] * 5 + [ctypes.c_int]
        L.orc_fill_normal.argtypes = [_i64p, _f64p, _f32p] + [ctypes.c_int64] * 5 + [ctypes.c_int]
        L.orc_fisher_replicates.argtypes = [
            _i64p, _i64p, ctypes.c_int, _i64p, ctypes.c_int, _f64p, ctypes.c_double,
            ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _f64p, _i64p, ctypes.c_int]
        L.orc_fisher_replicates.restype = ctypes.c_int64
        L.orc_rcont2_table.argtypes = [_i64p, ctypes.c_int, _i64p, ctypes.c_int, _f64p, _i64p, _i64p]
        L.orc_jump_matrices.argtypes = [ctypes.c_int, _i64p, _i64p]
        L.orc_skip.argtypes = [_i64p, ctypes.c_uint64]
        L.orc_create_streams.argtypes = [_i64p, ctypes.c_int64, _i64p, _i64p]
        L.orc_max_threads.restype = ctypes.c_int
        L.orc_box_muller.argtypes = [_i64p, _i64p, ctypes.c_int64, _f64p, _f64p]
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t) if a is not None else None


def _i64(a):
    a = np.ascontiguousarray(a, dtype=np.int64)
    return a


def max_threads() -> int:
    return lib().orc_max_threads()


def step(state6: np.ndarray) -> int:
    assert state6.dtype == np.int64 and state6.flags.c_contiguous
    return int(lib().orc_step(_p(state6, _i64p)))


def fill_real(cur, out, nrow, ncol, npad, g0, g1, mode, rate, threads=0):
    """_kernels.fill_real (_kernels.py:50-80); cur/out mutated in place."""
    assert cur.dtype == np.int64 and cur.flags.c_contiguous
    assert out.dtype == np.float64 and out.flags.c_contiguous
    lib().orc_fill_real(_p(cur, _i64p), _p(out, _f64p), nrow, ncol, npad, g0, g1,
                        int(mode), float(rate), int(threads))


def fill_integer(cur, out, nrow, ncol, npad, g0, g1, threads=0):
    """_kernels.fill_integer (_kernels.py:83-105)."""
    assert cur.dtype == np.int64 and out.dtype == np.int64
    lib().orc_fill_integer(_p(cur, _i64p), _p(out, _i64p), nrow, ncol, npad, g0, g1,
                           int(threads))


def fill_normal(cur, out, nrow, ncol, npad, g0, g1, threads=0):
    """_kernels.fill_normal (_kernels.py:108-166); out float64 or float32
    (float32 = the reference double rounded once, the GPU f32 anchor)."""
    assert cur.dtype == np.int64 and out.flags.c_contiguous
    if out.dtype == np.float64:
        lib().orc_fill_normal(_p(cur, _i64p), _p(out, _f64p), None, nrow, ncol, npad,
                              g0, g1, int(threads))
    elif out.dtype == np.float32:
        lib().orc_fill_normal(_p(cur, _i64p), None, _p(out, _f32p), nrow, ncol, npad,
                              g0, g1, int(threads))
    else:
        raise TypeError(out.dtype)


def fisher_replicates(cur, nrowt, ncolt, lf, threshold, reps, nitems, stats=None,
                      item_lo=0, item_counts=None, threads=0):
    """_kernels.fisher_replicates (_kernels.py:169-286) over items
    [item_lo, nitems); returns the hit count."""
    assert cur.dtype == np.int64 and cur.flags.c_contiguous
    nrowt = _i64(nrowt)
    ncolt = _i64(ncolt)
    lf = np.ascontiguousarray(lf, dtype=np.float64)
    if stats is not None:
        assert stats.dtype == np.float64
    if item_counts is not None:
        assert item_counts.dtype == np.int64
    return int(lib().orc_fisher_replicates(
        _p(cur, _i64p), _p(nrowt, _i64p), len(nrowt), _p(ncolt, _i64p), len(ncolt),
        _p(lf, _f64p), float(threshold), int(reps), int(item_lo), int(nitems),
        _p(stats, _f64p), _p(item_counts, _i64p), int(threads)))


def rcont2_table(nrowt, ncolt, lf, state):
    """_kernels.rcont2_table (_kernels.py:289-391); state mutated."""
    nrowt = _i64(nrowt)
    ncolt = _i64(ncolt)
    lf = np.ascontiguousarray(lf, dtype=np.float64)
    assert state.dtype == np.int64 and state.flags.c_contiguous
    mat = np.zeros((len(nrowt), len(ncolt)), dtype=np.int64)
    lib().orc_rcont2_table(_p(nrowt, _i64p), len(nrowt), _p(ncolt, _i64p), len(ncolt),
                           _p(lf, _f64p), _p(state, _i64p), _p(mat, _i64p))
    return mat


def jump_matrices(e):
    j1 = np.zeros(9, np.int64)
    j2 = np.zeros(9, np.int64)
    lib().orc_jump_matrices(int(e), _p(j1, _i64p), _p(j2, _i64p))
    return j1.reshape(3, 3), j2.reshape(3, 3)


def skip(state6, n):
    s = _i64(state6).copy()
    lib().orc_skip(_p(s, _i64p), int(n))
    return s


def create_streams(seed, n):
    """core.create_streams (core.py:222-235): returns (rows (n,6), next_seed)."""
    seed = _i64(seed)
    rows = np.empty((n, 6), np.int64)
    nxt = np.empty(6, np.int64)
    lib().orc_create_streams(_p(seed, _i64p), int(n), _p(rows, _i64p), _p(nxt, _i64p))
    return rows, tuple(int(x) for x in nxt)


def box_muller(z1, z2):
    """_kernels.py:147-152 on arbitrary draws (libm log/cos/sqrt)."""
    z1 = _i64(z1)
    z2 = _i64(z2)
    a = np.empty(len(z1))
    b = np.empty(len(z1))
    lib().orc_box_muller(_p(z1, _i64p), _p(z2, _i64p), len(z1), _p(a, _f64p), _p(b, _f64p))
    return a, b
