"""The drop-in at the reference's own seam: the UNMODIFIED reference package
(baseline/_ref, installed offline from /root/reference/pkg) run twice -- on its
numba `_kernels` and on paper_2201_06604_b200.reference_backend (libsfb.so on
the B200) -- through its public API.  Same outputs and stream states.
Skipped when baseline/_ref is not installed."""

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(os.path.join(REF, "streamforge")):
        pytest.skip("baseline/_ref (the installed reference) is not present")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/sfb_numba_cache")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import streamforge

    return streamforge


def both(ref, fn):
    """fn(streamforge) on the numba kernels, then on the B200 backend."""
    from paper_2201_06604_b200 import reference_backend

    a = fn(ref)
    undo = reference_backend.install(ref)
    try:
        b = fn(ref)
    finally:
        undo()
    return a, b


def fresh(ref, n):
    return ref.create_streams(ref.set_base_creator(), n)[0]


@pytest.mark.parametrize("kind,shape,grid,rate", [
    ("uniform", 8, (2, 2), 1.0), ("uniform", (64, 96), (8, 8), 1.0),
    ("uniform", (257, 300), (16, 16), 1.0), ("uniform-integer", (40, 70), (4, 10), 1.0),
    ("exponential", (33, 47), (4, 4), 0.7)])
def test_fills_bit_exact(ref, kind, shape, grid, rate):
    def run(sf):
        st = fresh(sf, grid[0] * grid[1])
        buf = sf.fill(st, sf.FillRequest(shape=shape, kind=kind, rate=rate,
                                         grid=sf.WorkGrid(*grid)))
        return buf.data.copy(), st.current.copy()

    (da, sa), (db, sb) = both(ref, run)
    assert np.array_equal(da, db)
    assert np.array_equal(sa, sb)


def test_normals_within_tolerance(ref):
    def run(sf):
        st = fresh(sf, 64)
        buf = sf.fill_normal(st, sf.FillRequest(shape=(60, 64), grid=sf.WorkGrid(4, 16)))
        return buf.data.copy(), st.current.copy()

    (da, sa), (db, sb) = both(ref, run)
    err = np.abs(da - db)
    assert ((err <= 4 * np.spacing(np.abs(da))) | (err <= 2.0 ** -60)).all()
    assert np.array_equal(sa, sb)


def test_fisher_sim_bit_exact(ref):
    from conftest import golden_arrays

    month = np.asarray(golden_arrays()["month"], np.int64)

    def run(sf):
        st = fresh(sf, 16)
        r = sf.fisher_sim(month, 2000, st, grid=sf.WorkGrid(4, 4), return_stats=True)
        return r.counts, r.p_value, r.statistics.copy(), st.current.copy()

    a, b = both(ref, run)
    assert a[0] == b[0] and a[1] == b[1]
    assert np.array_equal(a[2], b[2])
    assert np.array_equal(a[3], b[3])


def test_rcont2_bit_exact(ref):
    from conftest import golden_arrays

    month = np.asarray(golden_arrays()["month"], np.int64)

    def run(sf):
        state = np.array([12345] * 6, dtype=np.int64)
        tabs = [sf.rcont2(month.sum(1), month.sum(0), state) for _ in range(5)]
        return np.stack(tabs), state.copy()

    (ta, sa), (tb, sb) = both(ref, run)
    assert np.array_equal(ta, tb)
    assert np.array_equal(sa, sb)
