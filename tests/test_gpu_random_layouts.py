"""Randomised layouts through the C ABI (hypothesis): arbitrary matrix shapes,
work grids, padding, kinds and ARBITRARY item-range splits (shards of any size,
unaligned) -- every split composes to the single-launch result, which equals
the oracle bit for bit (uniform kinds) or within the normal contract.  This
exercises the quad, pair and generic kernels and their dispatch."""

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as hs

import paper_2201_06604_b200 as sf  # noqa: F401  (library load / device check)
from paper_2201_06604_b200.grid import launch_fill

import oracle_api as oa

pytestmark = pytest.mark.gpu


@hs.composite
def layouts(draw):
    kind = draw(hs.sampled_from(["uniform", "uniform-integer", "exponential", "normal",
                                 "normal32"]))
    g0 = draw(hs.integers(1, 9))
    g1 = draw(hs.integers(1, 12))
    if kind.startswith("normal") and g1 % 2:
        g1 += 1
    nrow = draw(hs.integers(1, 40))
    ncol = draw(hs.integers(1, 60))
    npad = ncol + draw(hs.sampled_from([0, 0, 0, 1, 2, 3, 8]))
    # split the unit range (items, or pairs for normals) at random points
    nunits = g0 * g1 // (2 if kind.startswith("normal") else 1)
    cuts = sorted(set(draw(hs.lists(hs.integers(0, nunits), max_size=4))) | {0, nunits})
    rate = draw(hs.sampled_from([1.0, 0.37, 2.5]))
    return kind, g0, g1, nrow, ncol, npad, cuts, rate


def _device_fill(kind, g0, g1, nrow, ncol, npad, cuts, rate):
    import torch

    n = g0 * g1
    cur = torch.from_numpy(oa.fresh_states(n)).cuda()
    dt = {"uniform-integer": torch.int64, "normal32": torch.float32}.get(kind, torch.float64)
    out = torch.zeros((nrow, npad), dtype=dt, device="cuda")
    k = "normal" if kind.startswith("normal") else kind
    scale = 2 if k == "normal" else 1
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        if hi > lo:
            launch_fill(k, cur, n, out, nrow, ncol, npad, g0, g1, rate=rate,
                        item_lo=lo * scale, item_hi=hi * scale)
    torch.cuda.synchronize()
    return out.cpu().numpy(), cur.cpu().numpy()


@settings(max_examples=150, deadline=None, suppress_health_check=list(HealthCheck))
@given(layouts())
def test_random_layouts_and_splits_match_oracle(lay):
    kind, g0, g1, nrow, ncol, npad, cuts, rate = lay
    got, states = _device_fill(*lay)
    ref_states = oa.fresh_states(g0 * g1)
    k = "normal" if kind.startswith("normal") else kind
    ref = oa.fill(k, ref_states, (nrow, ncol), (g0, g1), npad=npad, rate=rate)
    assert np.array_equal(states, ref_states), lay
    if k != "normal":
        assert np.array_equal(got, ref), lay
        return
    if kind == "normal32":
        r32 = ref.astype(np.float32)
        d = np.abs(got.astype(np.float64) - r32.astype(np.float64))
        assert (d <= np.spacing(np.abs(r32)).astype(np.float64)).all(), lay
    else:
        err = np.abs(got - ref)
        assert ((err <= 4 * np.spacing(np.abs(ref))) | (err <= 2.0 ** -60)).all(), lay


@hs.composite
def fisher_cases(draw):
    nr = draw(hs.integers(1, 6))
    nc = draw(hs.integers(1, 6))
    if nr * nc < 2:
        nc = 2
    scale = draw(hs.sampled_from([2, 10, 60, 400]))
    table = np.array(draw(hs.lists(hs.integers(0, scale), min_size=nr * nc, max_size=nr * nc)),
                     dtype=np.int64).reshape(nr, nc)
    if table.sum() == 0:
        table[0, 0] = 1
    g0 = draw(hs.integers(1, 8))
    g1 = draw(hs.integers(1, 8))
    reps = draw(hs.integers(1, 40))
    cuts = sorted(set(draw(hs.lists(hs.integers(0, g0 * g1), max_size=3))) | {0, g0 * g1})
    memo = draw(hs.sampled_from(["0", "1"]))
    return table, g0, g1, reps, cuts, memo


@settings(max_examples=120, deadline=None, suppress_health_check=list(HealthCheck))
@given(fisher_cases())
def test_random_fisher_tables_and_splits_match_oracle(case):
    """Random margins (zeros, degenerate rows/columns, wide ranges), grids,
    replicate counts and item splits, memo on/off: counts, statistics and
    final states bit for bit."""
    import os

    import torch

    from paper_2201_06604_b200 import _lib

    table, g0, g1, reps, cuts, memo = case
    n = g0 * g1
    rm, cm = table.sum(1), table.sum(0)
    lf = oa.lf_table(int(table.sum()))
    thr = oa.relaxed(oa.logfact_sum(table))
    cur = torch.from_numpy(oa.fresh_states(n)).cuda()
    stats = torch.empty(n * reps, dtype=torch.float64, device="cuda")
    count = torch.zeros(1, dtype=torch.int64, device="cuda")
    os.environ["SFB_FISHER_MEMO"] = memo
    try:
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            if hi > lo:
                _lib.check(_lib.lib().sfb_fisher_replicates(
                    _lib.dptr(cur), n, _lib.ptr(np.ascontiguousarray(rm)), len(rm),
                    _lib.ptr(np.ascontiguousarray(cm)), len(cm), _lib.ptr(lf, _lib._f64p),
                    len(lf), thr, reps, lo, hi, _lib.dptr(stats[lo * reps:]), None,
                    _lib.dptr(count), 0, _lib.stream_handle()))
        torch.cuda.synchronize()
    finally:
        os.environ.pop("SFB_FISHER_MEMO", None)
    ref_states = oa.fresh_states(n)
    ref_stats = np.empty(n * reps)
    from oracle import oracle as orc

    rc = orc.fisher_replicates(ref_states, rm, cm, lf, thr, reps, n, ref_stats)
    assert int(count.item()) == rc, case
    assert np.array_equal(stats.cpu().numpy(), ref_stats), case
    assert np.array_equal(cur.cpu().numpy(), ref_states), case
