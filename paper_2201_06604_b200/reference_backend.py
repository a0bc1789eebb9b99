"""`streamforge._kernels`-compatible backend over the C ABI (the drop-in seam).

The reference's only native boundary is its `_kernels` module
(/root/reference/pkg/src/streamforge/_kernels.py): numba functions that take
host numpy arrays, mutate the stream states `cur` and the output `out` in
place and return.  This module provides the same six functions with the same
signatures and in-place semantics, backed by libsfb.so (include/sfb.h) -- so
the UNMODIFIED reference package (grid.py, distributions.py, fisher.py) runs
on the B200 when its `_kernels` is swapped:

    import streamforge
    from paper_2201_06604_b200 import reference_backend
    reference_backend.install(streamforge)      # patches streamforge._kernels

Every call uploads the host arrays, runs the kernel and copies the results back
into them (that is the numba contract); `paper_2201_06604_b200` itself keeps
states and outputs in HBM between calls instead.  tests/test_reference_backend.py
runs the installed reference package both ways and compares the results.
"""

from __future__ import annotations

import numpy as np

from . import _lib

F64 = 0  # SFB_F64


def _dev(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _back(host, dev):
    import torch

    if host.flags.c_contiguous and host.size == dev.numel():
        torch.from_numpy(host).view(dev.dtype).reshape(dev.shape).copy_(dev)  # one copy
    else:
        host[...] = dev.cpu().numpy().reshape(host.shape)


def max_threads():  # _kernels.py:25-26
    return 1


def set_threads(n):  # _kernels.py:29-30 -- thread counts never change results
    return None


def fill_real(cur, out, nrow, ncol, npad, g0, g1n, mode, rate):  # _kernels.py:50-80
    _lib.require_device()
    dcur, dout = _dev(cur), _dev(out)
    _lib.check(_lib.lib().sfb_fill_real(
        _lib.dptr(dcur), cur.shape[0], _lib.dptr(dout), nrow, ncol, npad, g0, g1n, int(mode),
        float(rate), 0, g0 * g1n, 0, _lib.stream_handle()))
    _back(cur, dcur)
    _back(out, dout)


def fill_integer(cur, out, nrow, ncol, npad, g0, g1n):  # _kernels.py:83-105
    _lib.require_device()
    dcur, dout = _dev(cur), _dev(out)
    _lib.check(_lib.lib().sfb_fill_integer(
        _lib.dptr(dcur), cur.shape[0], _lib.dptr(dout), nrow, ncol, npad, g0, g1n, 0, g0 * g1n,
        0, _lib.stream_handle()))
    _back(cur, dcur)
    _back(out, dout)


def fill_normal(cur, out, nrow, ncol, npad, g0, g1n):  # _kernels.py:108-166
    _lib.require_device()
    dcur, dout = _dev(cur), _dev(out)
    _lib.check(_lib.lib().sfb_fill_normal(
        _lib.dptr(dcur), cur.shape[0], _lib.dptr(dout), F64, nrow, ncol, npad, g0, g1n, 0,
        g0 * g1n, 0, _lib.stream_handle()))
    _back(cur, dcur)
    _back(out, dout)


def fisher_replicates(cur, nrowt, ncolt, lf, threshold, reps, nitems, stats,
                      want_stats):  # _kernels.py:169-286
    import torch

    _lib.require_device()
    dcur = _dev(cur)
    count = torch.empty(1, dtype=torch.int64, device="cuda")
    dstats = torch.empty(max(1, nitems * reps), dtype=torch.float64, device="cuda") \
        if want_stats else None
    rm = np.ascontiguousarray(nrowt, np.int64)
    cm = np.ascontiguousarray(ncolt, np.int64)
    lfc = np.ascontiguousarray(lf, np.float64)
    _lib.check(_lib.lib().sfb_fisher_replicates(
        _lib.dptr(dcur), cur.shape[0], _lib.ptr(rm), len(rm), _lib.ptr(cm), len(cm),
        _lib.ptr(lfc, _lib._f64p), len(lfc), float(threshold), int(reps), 0, int(nitems),
        None if dstats is None else _lib.dptr(dstats), None, _lib.dptr(count), 1,
        _lib.stream_handle()))
    _back(cur, dcur)
    if want_stats:
        _back(stats[: nitems * reps], dstats[: nitems * reps])
    return int(count.item())


def rcont2_table(nrowt, ncolt, lf, state):  # _kernels.py:289-391
    import torch

    _lib.require_device()
    rm = np.ascontiguousarray(nrowt, np.int64)
    cm = np.ascontiguousarray(ncolt, np.int64)
    lfc = np.ascontiguousarray(lf, np.float64)
    dstate = _dev(np.asarray(state, np.int64).reshape(6))
    dmat = torch.zeros((len(rm), len(cm)), dtype=torch.int64, device="cuda")
    _lib.check(_lib.lib().sfb_rcont2_table(
        _lib.ptr(rm), len(rm), _lib.ptr(cm), len(cm), _lib.ptr(lfc, _lib._f64p), len(lfc),
        _lib.dptr(dstate), _lib.dptr(dmat), _lib.stream_handle()))
    state[...] = dstate.cpu().numpy().reshape(np.shape(state))
    return dmat.cpu().numpy()


FUNCTIONS = ("max_threads", "set_threads", "fill_real", "fill_integer", "fill_normal",
             "fisher_replicates", "rcont2_table")


def install(streamforge_module):
    """Point `streamforge._kernels` at this backend; returns an undo callable."""
    import importlib

    kernels = importlib.import_module(streamforge_module.__name__ + "._kernels")
    saved = {name: getattr(kernels, name) for name in FUNCTIONS if hasattr(kernels, name)}
    this = globals()
    for name in FUNCTIONS:
        setattr(kernels, name, this[name])

    def undo():
        for name, fn in saved.items():
            setattr(kernels, name, fn)

    return undo
