"""Test helpers: the reference's public-API semantics driven through the CPU
oracle (grid.py:112-144, distributions.py:31-52, fisher.py:118-164 restated
over oracle/).  Test infrastructure only."""

from __future__ import annotations

import numpy as np
from scipy.special import gammaln

from oracle import oracle as orc

DEFAULT_SEED = (12345,) * 6


def fresh_states(n, seed=DEFAULT_SEED):
    rows, _ = orc.create_streams(seed, n)
    return rows


def dims(shape):
    """FillRequest.dims (distributions.py:31-52) for valid shapes."""
    if isinstance(shape, int):
        return 1, shape
    shape = tuple(int(x) for x in shape)
    if len(shape) == 1:
        return 1, shape[0]
    return shape


def fill(kind, states, shape, grid, npad=None, rate=1.0, out_dtype=None, threads=0):
    """run_grid (grid.py:112-144) on the oracle; states mutated in place."""
    nrow, ncol = dims(shape)
    npad = ncol if npad is None else npad
    g0, g1 = grid
    if kind == "uniform-integer":
        data = np.zeros((nrow, npad), np.int64)
        orc.fill_integer(states, data.ravel(), nrow, ncol, npad, g0, g1, threads)
    elif kind in ("uniform", "exponential"):
        data = np.zeros((nrow, npad), np.float64)
        orc.fill_real(states, data.ravel(), nrow, ncol, npad, g0, g1,
                      0 if kind == "uniform" else 1, rate, threads)
    elif kind == "normal":
        data = np.zeros((nrow, npad), out_dtype or np.float64)
        orc.fill_normal(states, data.ravel(), nrow, ncol, npad, g0, g1, threads)
    else:
        raise ValueError(kind)
    return data


def lf_table(total):
    """fisher.log_factorial_table (fisher.py:70-72)."""
    return gammaln(np.arange(total + 1, dtype=np.float64) + 1.0)


def logfact_sum(table):
    """fisher.logfact_sum (fisher.py:75-80)."""
    return float(-gammaln(np.asarray(table, dtype=np.float64) + 1.0).sum())


def relaxed(t):
    """fisher.relaxed_threshold (fisher.py:113-115)."""
    return t + 1e-7 * abs(t)


def fisher(table, n, states, grid, return_stats=False, threads=0):
    """fisher_sim (fisher.py:118-164) on the oracle."""
    table = np.asarray(table, dtype=np.int64)
    g0, g1 = grid
    size = g0 * g1
    sim_num = -(-n // size) * size
    reps = sim_num // size
    thr = logfact_sum(table)
    lf = lf_table(int(table.sum()))
    stats = np.empty(sim_num, np.float64) if return_stats else None
    counts = orc.fisher_replicates(states, table.sum(axis=1), table.sum(axis=0), lf,
                                   relaxed(thr), reps, size, stats, threads=threads)
    return dict(threshold=thr, sim_num=sim_num, counts=counts,
                p_value=(1 + counts) / (sim_num + 1), statistics=stats)
