"""GRF pipeline against the CPU restatement of the
reference (oracle/oracle_grf.py: scipy kv, pdist, LAPACK dpotrf, numpy) and
the reference's own behavioural tests (tests/test_grf.py, test_acceptance.py
09-11 of /root/reference/pkg), within their tolerances."""

import math

import numpy as np
import pytest
from scipy.special import kv

import paper_2201_06604_b200 as sf
from oracle import oracle_grf as og
from paper_2201_06604_b200 import _lib
from paper_2201_06604_b200.errors import (InvalidArgumentError, InvalidParamsError,
                                          InvalidShapesError, NotPositiveDefiniteError)
from paper_2201_06604_b200.grf import BatchedMatrix, DiagBatch

import oracle_api as oa


# ------------------------------------------------------------------ CPU
def test_host_bessel_k_against_scipy():
    """csrc/bessel_k.cuh (the device K_nu) on the host vs scipy.special.kv."""
    rng = np.random.default_rng(1)
    nus = np.concatenate([rng.uniform(0.05, 4.0, 3000), [0.5, 1.0, 1.5, 2.0, 2.5] * 20])
    xs = np.exp(rng.uniform(math.log(1e-8), math.log(600.0), len(nus)))
    xs[:300] = rng.uniform(1.9, 2.1, 300)  # the method switch at x = 2
    f = _lib.lib().sfb_host_bessel_k
    got = np.array([f(float(a), float(b)) for a, b in zip(nus, xs)])
    ref = kv(nus, xs)
    ok = ref > 0
    rel = np.abs(got[ok] - ref[ok]) / ref[ok]
    assert rel.max() < 5e-13, rel.max()
    # closed form K_1/2(x) = sqrt(pi / 2x) e^-x (reference tests/test_grf.py:19-24)
    for x in (0.25, 1.0, 3.0):
        assert abs(f(0.5, x) - math.sqrt(math.pi / (2 * x)) * math.exp(-x)) < 1e-14
    assert round(f(1.0, 1.0), 7) == 0.6019072


def test_params_and_grid_validation():
    with pytest.raises(InvalidParamsError):
        sf.MaternParams(shape=-1.0, range=1.0, variance=1.0)
    with pytest.raises(InvalidParamsError):
        sf.MaternParams(shape=1.0, range=1.0, variance=1.0, aniso_ratio=0.5)
    with pytest.raises(InvalidParamsError):
        sf.MaternParams.from_row([1.0, 2.0, 3.0])
    with pytest.raises(InvalidArgumentError):
        sf.GridSpec(0, 2, 1.0)
    with pytest.raises(InvalidArgumentError):
        sf.GridSpec(2, 2, 0.0)
    assert np.array_equal(sf.GridSpec(2, 2, 2.0, origin=(10.0, 20.0)).cell_coords(),
                          [[11.0, 21.0], [13.0, 21.0], [11.0, 23.0], [13.0, 23.0]])
    assert np.array_equal(sf.GridSpec(7, 5, 0.3, origin=(1.0, -2.0)).cell_coords(),
                          og.grid_coords(7, 5, 0.3, (1.0, -2.0)))


def test_domain_and_shape_errors_before_any_device_work():
    with pytest.raises(InvalidArgumentError):
        sf.bessel_k(0.0, 1.0)
    with pytest.raises(InvalidArgumentError):
        sf.bessel_k(1.0, 0.0)
    with pytest.raises(InvalidArgumentError):
        sf.bessel_k(1.0, np.array([1.0, -2.0]))
    lmat = BatchedMatrix(np.eye(2), 1)
    diag = DiagBatch(np.ones((1, 2)))
    with pytest.raises(InvalidShapesError):
        sf.multiply_lower_diag_batch(lmat, diag, np.ones(3))
    with pytest.raises(InvalidShapesError):
        sf.multiply_lower_diag_batch(lmat, DiagBatch(np.ones((1, 3))), np.ones(2))
    with pytest.raises(InvalidArgumentError):
        sf.multiply_lower_diag_batch(lmat, diag, np.ones(2), transform="square")
    with pytest.raises(InvalidShapesError):
        BatchedMatrix(np.ones((3, 2)), 2)
    with pytest.raises(InvalidParamsError):
        sf.simulate_grf([], sf.GridSpec(2, 2, 1.0), 1, sf.create_streams(
            sf.set_base_creator(), 4)[0], sf.WorkGrid(2, 2))
    with pytest.raises(InvalidArgumentError):
        sf.simulate_grf([sf.MaternParams(1.0, 2.0, 1.0)], sf.GridSpec(2, 2, 1.0), 0,
                        sf.create_streams(sf.set_base_creator(), 4)[0], sf.WorkGrid(2, 2))


# ------------------------------------------------------------------ GPU
PARAMS = [(1.0, 2.0, 1.0, 1.0, 0.0), (1.5, 3.0, 2.0, 2.0, 0.5), (0.5, 6.0, 1.5, 1.0, 0.0),
          (2.0, 10.0, 1.0, 1.5, 1.0), (0.3, 1.2, 0.7, 3.0, -0.7)]


@pytest.mark.gpu
def test_bessel_k_device_against_scipy():
    rng = np.random.default_rng(2)
    xs = np.exp(rng.uniform(math.log(1e-6), math.log(300.0), 20000))
    for nu in (0.3, 0.5, 1.0, 1.7, 2.5, 3.9):
        got = sf.bessel_k(nu, xs)
        ref = kv(nu, xs)
        assert (np.abs(got - ref) <= 5e-13 * ref).all(), nu
    for nu in (0.5, 1.3, 1.7):  # reference tests/test_grf.py:29-35
        for x in (0.3, 1.0, 4.0):
            lhs = sf.bessel_k(nu + 1.0, x)
            rhs = sf.bessel_k(abs(nu - 1.0), x) + (2 * nu / x) * sf.bessel_k(nu, x)
            assert abs(lhs - rhs) < 1e-9 * abs(rhs)


@pytest.mark.gpu
def test_matern_correlation_against_scipy_and_closed_forms():
    d = np.concatenate([[0.0], np.linspace(1e-6, 40.0, 5000)])
    for p in PARAMS:
        got = sf.matern_correlation(sf.MaternParams(*p), d)
        ref = og.matern_correlation(p, d)
        assert got[0] == 1.0
        assert np.allclose(got, ref, rtol=1e-12, atol=1e-300)
    p = sf.MaternParams(shape=0.5, range=1.7, variance=1.0)  # acceptance 09
    dd = np.linspace(0.01, 5.0, 50)
    assert np.allclose(sf.matern_correlation(p, dd), np.exp(-2.0 * dd / 1.7), rtol=1e-10, atol=0)
    for kappa in (0.5, 1.0, 2.0):
        c = float(sf.matern_correlation(sf.MaternParams(kappa, 2.5, 1.0), np.array([2.5]))[0])
        assert abs(c - 0.14) < 0.02


@pytest.mark.gpu
@pytest.mark.parametrize("nx,ny,cell", [(4, 3, 1.0), (5, 5, 0.7), (13, 7, 0.45)])
def test_matern_cov_grid_against_oracle(nx, ny, cell):
    grid = sf.GridSpec(nx, ny, cell)
    cov = sf.matern_cov([sf.MaternParams(*p) for p in PARAMS], grid)
    ref = og.matern_cov(PARAMS, og.grid_coords(nx, ny, cell))
    assert np.allclose(cov.data, ref, rtol=1e-12, atol=1e-15)
    for b, p in enumerate(PARAMS):
        blk = cov.block(b)
        assert np.array_equal(blk, blk.T)  # exactly symmetric
        assert np.array_equal(np.diagonal(blk), np.full(grid.ncell, p[2]))  # exact variance


@pytest.mark.gpu
def test_matern_cov_arbitrary_coords_against_oracle():
    rng = np.random.default_rng(7)
    coords = rng.uniform(0, 10, size=(300, 2))
    cov = sf.matern_cov([sf.MaternParams(*p) for p in PARAMS], coords)
    ref = og.matern_cov(PARAMS, coords)
    assert np.allclose(cov.data, ref, rtol=1e-12, atol=1e-15)
    for b in range(len(PARAMS)):
        assert np.array_equal(cov.block(b), cov.block(b).T)
    # reference tests/test_grf.py:100-115: anisotropy and a direct entry
    c = sf.matern_cov([sf.MaternParams(1.0, 2.0, 1.0, 4.0, 0.0)],
                      np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]])).block(0)
    assert c[0, 1] > c[0, 2]
    p = sf.MaternParams(1.2, 2.0, 1.7)
    c = sf.matern_cov([p], np.array([[0.0, 0.0], [3.0, 4.0]])).block(0)
    assert abs(c[0, 1] - 1.7 * float(sf.matern_correlation(p, np.array([5.0]))[0])) < 1e-14
    g = sf.GridSpec(6, 4, 1.0)
    a = sf.matern_cov([sf.MaternParams(1.0, 2.0, 1.0, 1.0, 0.0)], g).block(0)
    b = sf.matern_cov([sf.MaternParams(1.0, 2.0, 1.0, 1.0, 0.9)], g).block(0)
    assert np.allclose(a, b, rtol=0, atol=1e-12)


@pytest.mark.gpu
def test_chol_batch_against_oracle_and_hand_cases():
    lm, dg = sf.chol_batch(BatchedMatrix(np.eye(3), 1))
    assert np.array_equal(lm.block(0), np.eye(3)) and np.array_equal(dg.data, np.ones((1, 3)))
    lm, dg = sf.chol_batch(BatchedMatrix(np.array([[4.0, 2.0], [2.0, 3.0]]), 1))
    assert np.allclose(lm.block(0), [[1.0, 0.0], [0.5, 1.0]], rtol=0, atol=1e-14)
    assert np.allclose(dg.data[0], [4.0, 2.0], rtol=0, atol=1e-14)
    rng = np.random.default_rng(3)  # acceptance 10: 512 x 512 round trip
    coords = rng.uniform(0, 10, size=(512, 2))
    cov = sf.matern_cov([sf.MaternParams(1.5, 3.0, 2.0)], coords)
    lmat, diag = sf.chol_batch(cov)
    rebuilt = lmat.block(0) @ np.diag(diag.data[0]) @ lmat.block(0).T
    assert np.abs(rebuilt - cov.block(0)).max() < 1e-8 * np.abs(cov.block(0)).max()
    rl, rd = og.chol_batch(cov.data, 1)
    assert np.allclose(lmat.data, rl, rtol=1e-8, atol=1e-10)
    assert np.allclose(diag.data, rd, rtol=1e-8, atol=1e-12)


@pytest.mark.gpu
def test_not_positive_definite_names_batch_and_pivot():
    data = np.vstack([np.eye(2), np.array([[1.0, 2.0], [2.0, 1.0]])])
    with pytest.raises(NotPositiveDefiniteError) as exc:
        sf.chol_batch(BatchedMatrix(data, 2))
    assert exc.value.batch == 1 and exc.value.pivot == 2  # LAPACK dpotrf info


@pytest.mark.gpu
@pytest.mark.parametrize("n,nb", [(1, 1), (63, 2), (64, 1), (65, 3), (129, 2), (333, 2), (600, 1)])
def test_chol_batch_tiles_odd_and_ragged_sizes(n, nb):
    """csrc/chol.cu on sizes around its 64-tile grid (ragged last tile; odd n:
    the synchronous loader) against the oracle (scipy LAPACK), grf.py:190-208."""
    rng = np.random.default_rng(n)
    blocks = []
    for _ in range(nb):
        a = rng.standard_normal((n, n))
        blocks.append(a @ a.T + n * np.eye(n))  # SPD, well conditioned
    data = np.vstack(blocks)
    lmat, diag = sf.chol_batch(BatchedMatrix(data, nb))
    rl, rd = og.chol_batch(data, nb)
    assert np.allclose(lmat.data, rl, rtol=1e-10, atol=1e-12)
    assert np.allclose(diag.data, rd, rtol=1e-10, atol=1e-12)
    for b in range(nb):
        lb = lmat.block(b)
        assert np.array_equal(np.triu(lb, 1), np.zeros((n, n)))
        assert np.array_equal(np.diag(lb), np.ones(n))


@pytest.mark.gpu
@pytest.mark.parametrize("panel,split", [(1, 1), (2, 1), (3, 0), (8, 0), (32, 1)])
def test_chol_batch_schedules_agree(monkeypatch, panel, split):
    """Every super-panel width / stream split of the look-ahead schedule
    (SFB_CHOL_PANEL, SFB_CHOL_SPLIT) factors to the oracle's L and D: the
    fused panel kernel in both modes, the delayed and panel-local updates."""
    monkeypatch.setenv("SFB_CHOL_PANEL", str(panel))
    monkeypatch.setenv("SFB_CHOL_SPLIT", str(split))
    n, nb = 700, 2
    rng = np.random.default_rng(panel * 10 + split)
    blocks = []
    for _ in range(nb):
        a = rng.standard_normal((n, n))
        blocks.append(a @ a.T + n * np.eye(n))
    data = np.vstack(blocks)
    lmat, diag = sf.chol_batch(BatchedMatrix(data, nb))
    rl, rd = og.chol_batch(data, nb)
    assert np.allclose(lmat.data, rl, rtol=1e-10, atol=1e-12)
    assert np.allclose(diag.data, rd, rtol=1e-10, atol=1e-12)


@pytest.mark.gpu
def test_chol_batch_default_schedule_with_bulk_updates():
    """n = 1500 (24 tiles, three 8-tile super-panels) on the default
    schedule: the per-column look-ahead updates on their own stream and the
    bulk update split into near / far columns all run; L and D match the
    oracle (LAPACK)."""
    n, nb = 1500, 2
    rng = np.random.default_rng(1500)
    blocks = []
    for _ in range(nb):
        a = rng.standard_normal((n, n))
        blocks.append(a @ a.T + n * np.eye(n))
    data = np.vstack(blocks)
    lmat, diag = sf.chol_batch(BatchedMatrix(data, nb))
    rl, rd = og.chol_batch(data, nb)
    assert np.allclose(lmat.data, rl, rtol=1e-10, atol=1e-12)
    assert np.allclose(diag.data, rd, rtol=1e-10, atol=1e-12)


@pytest.mark.gpu
def test_chol_batch_concurrent_threads_and_streams():
    """Two host threads factor different batches on their own CUDA streams at
    once (the per-device look-ahead streams, events and scratch are shared
    under a lock): each result equals the same call made alone."""
    import threading

    import torch

    rng = np.random.default_rng(21)
    mats = []
    for n in (300, 515):
        a = rng.standard_normal((2 * n, n))
        blocks = [a[:n] @ a[:n].T + n * np.eye(n), a[n:] @ a[n:].T + n * np.eye(n)]
        mats.append(BatchedMatrix(np.vstack(blocks), 2))
    alone = [sf.chol_batch(m) for m in mats]
    alone = [(lm.data.copy(), dg.data.copy()) for lm, dg in alone]
    out = [None, None]

    def work(q):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(3):
                lm, dg = sf.chol_batch(mats[q])
            s.synchronize()
            out[q] = (lm.data, dg.data)

    ts = [threading.Thread(target=work, args=(q,)) for q in (0, 1)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for q in (0, 1):
        assert np.array_equal(out[q][0], alone[q][0])
        assert np.array_equal(out[q][1], alone[q][1])


@pytest.mark.gpu
def test_not_positive_definite_pivot_in_a_later_tile():
    """The first failing minor lies past the first 64-tile (LAPACK info = its
    order); the other blocks of the batch are unaffected by the failure."""
    n = 150
    rng = np.random.default_rng(11)
    a = rng.standard_normal((n, n))
    good = a @ a.T + n * np.eye(n)
    bad = good.copy()
    bad[100:, 100:] -= 1e6 * np.eye(n - 100)  # minor of order 101 is negative
    with pytest.raises(NotPositiveDefiniteError) as exc:
        sf.chol_batch(BatchedMatrix(np.vstack([good, bad, good]), 3))
    assert exc.value.batch == 1 and exc.value.pivot == 101


@pytest.mark.gpu
def test_multiply_lower_diag_batch_many_realisations_against_numpy():
    """R = 11 (the 8-column passes plus a remainder), Z shared and per block."""
    rng = np.random.default_rng(5)
    n, nb, r = 97, 3, 11
    lm = np.tril(rng.standard_normal((nb, n, n)), -1) + np.eye(n)
    d = rng.uniform(0.5, 2.0, (nb, n))
    for zrows in (n, nb * n):
        z = rng.standard_normal((zrows, r))
        for tr in ("sqrt", "identity"):
            out = sf.multiply_lower_diag_batch(BatchedMatrix(lm.reshape(nb * n, n), nb),
                                               DiagBatch(d), z, transform=tr)
            for b in range(nb):
                zb = z if zrows == n else z[b * n:(b + 1) * n]
                s = np.sqrt(d[b]) if tr == "sqrt" else d[b]
                ref = lm[b] @ (s[:, None] * zb)
                assert np.allclose(out.block(b), ref, rtol=1e-12, atol=1e-12)


@pytest.mark.gpu
def test_multiply_lower_diag_batch_cases():
    out = sf.multiply_lower_diag_batch(BatchedMatrix(np.eye(3), 1), DiagBatch(np.ones((1, 3))),
                                       np.arange(6.0).reshape(3, 2))
    assert np.array_equal(out.block(0), np.arange(6.0).reshape(3, 2))
    out = sf.multiply_lower_diag_batch(BatchedMatrix(np.array([[1.0, 0.0], [0.5, 1.0]]), 1),
                                       DiagBatch(np.array([[4.0, 2.0]])), np.array([1.0, 1.0]))
    assert np.allclose(out.block(0).ravel(), [2.0, 1.0 + math.sqrt(2.0)], rtol=0, atol=1e-14)
    out = sf.multiply_lower_diag_batch(BatchedMatrix(np.eye(2), 1),
                                       DiagBatch(np.array([[4.0, 9.0]])), np.ones(2),
                                       transform="identity")
    assert np.array_equal(out.block(0).ravel(), [4.0, 9.0])
    out = sf.multiply_lower_diag_batch(BatchedMatrix(np.vstack([np.eye(2), np.eye(2)]), 2),
                                       DiagBatch(np.ones((2, 2))), np.arange(4.0)[:, None])
    assert np.array_equal(out.block(0).ravel(), [0.0, 1.0])
    assert np.array_equal(out.block(1).ravel(), [2.0, 3.0])


@pytest.mark.gpu
def test_simulate_grf_against_oracle_with_the_same_normals():
    """The whole pipeline vs the CPU restatement fed with the oracle's normals
    from the same streams (the device normals are <= 4 ulp from them)."""
    nx, ny, r = 9, 7, 5
    params = PARAMS[:3]
    n, nb = nx * ny, len(params)
    st = sf.create_streams(sf.set_base_creator(), 16)[0]
    fields = sf.simulate_grf([sf.MaternParams(*p) for p in params], sf.GridSpec(nx, ny, 1.0), r,
                             st, sf.WorkGrid(4, 4))
    ref_st = oa.fresh_states(16)
    z = oa.fill("normal", ref_st, (nb * n, r), (4, 4))
    ref = og.simulate(params, nx, ny, 1.0, z)
    assert fields.shape == (nb, r, ny, nx)
    assert np.allclose(fields, ref, rtol=1e-9, atol=1e-11)
    assert np.array_equal(st.current, ref_st)


@pytest.mark.gpu
def test_simulate_grf_reference_properties():
    """reference tests/test_grf.py:221-239 and test_acceptance.py:210-245."""
    grid = sf.GridSpec(5, 4, 1.0)
    params = [sf.MaternParams(1.0, 2.0, 1.0), sf.MaternParams(0.5, 3.0, 2.0)]

    def fresh(n):
        return sf.create_streams(sf.set_base_creator(), n)[0]

    a = sf.simulate_grf(params, grid, 3, fresh(16), sf.WorkGrid(4, 4))
    b = sf.simulate_grf(params, grid, 3, fresh(16), sf.WorkGrid(4, 4))
    assert a.shape == (2, 3, 4, 5) and np.array_equal(a, b)
    g4 = sf.GridSpec(4, 4, 1.0)
    base = sf.simulate_grf([sf.MaternParams(1.0, 2.0, 1.0)], g4, 2, fresh(16), sf.WorkGrid(4, 4))
    scaled = sf.simulate_grf([sf.MaternParams(1.0, 2.0, 4.0)], g4, 2, fresh(16),
                             sf.WorkGrid(4, 4))
    assert np.allclose(scaled, 2.0 * base, rtol=1e-12, atol=0)
    # acceptance 11: variance and correlation recovery over 2000 realisations
    sigma2 = 2.0
    p = sf.MaternParams(shape=1.0, range=2.5, variance=sigma2)
    g10 = sf.GridSpec(10, 10, 1.0)
    fields = sf.simulate_grf([p], g10, 2000, fresh(64), sf.WorkGrid(8, 8))
    flat = fields[0].reshape(2000, g10.ncell)
    se_var = sigma2 * math.sqrt(2.0 / 2000)
    for cell in (0, 13, 47, 68, 99):
        assert abs(float((flat[:, cell] ** 2).mean()) - sigma2) < 5 * se_var
    cov = sf.matern_cov([p], g10).block(0)
    for i, j in ((0, 1), (0, 5), (44, 47)):
        se = math.sqrt((sigma2 * sigma2 + cov[i, j] ** 2) / 2000)
        assert abs(float((flat[:, i] * flat[:, j]).mean()) - cov[i, j]) < 5 * se
    # the full-size batch of acceptance 11: four 5130 x 5130 blocks
    big = sf.GridSpec(90, 57, 1.0)
    batch = [sf.MaternParams(1.0, 8.0, 1.0), sf.MaternParams(1.5, 12.0, 2.0, 2.0, 0.5),
             sf.MaternParams(0.5, 6.0, 1.5), sf.MaternParams(2.0, 10.0, 1.0, 1.5, 1.0)]
    fields = sf.simulate_grf(batch, big, 2, fresh(64), sf.WorkGrid(8, 8))
    assert fields.shape == (4, 2, 57, 90) and np.isfinite(fields).all()
