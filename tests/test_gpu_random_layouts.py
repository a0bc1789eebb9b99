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
