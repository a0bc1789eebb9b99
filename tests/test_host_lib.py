"""CPU tests of the product's host half and of the device arithmetic run on the
host: libsfb.so loads and exports every symbol of include/sfb.h, the uint32
MRG31k3p formulation equals the int64 reference step, the glibc exp port is
bit-exact against libm, the stream arithmetic / stream files match the
reference-generated goldens, and the API validates like the reference."""

import ctypes
import ctypes.util
import io
import math
import os
import re
import struct

import numpy as np
import pytest

import paper_2201_06604_b200 as sf
from paper_2201_06604_b200 import _lib
from paper_2201_06604_b200.errors import (
    CorruptStreamFileError,
    DeviceError,
    InsufficientStreamsError,
    InvalidArgumentError,
    InvalidGridError,
    InvalidMarginsError,
    InvalidRateError,
    InvalidSeedError,
)
from paper_2201_06604_b200.fisher import (
    ContingencyTable,
    log_factorial_table,
    relaxed_threshold,
    sim_num_for,
)

from conftest import PRINTED_STREAM_MATRIX, ROOT, has_gpu, sha
from oracle import oracle as orc


def test_library_exports_every_header_symbol():
    header = open(os.path.join(ROOT, "include", "sfb.h")).read()
    declared = set(re.findall(r"\b(sfb_[a-z0-9_]+)\s*\(", header))
    assert declared == set(_lib.EXPORTED)
    L = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared:
        assert hasattr(L, name), name
    assert _lib.lib().sfb_version() >= 100


def test_sm100a_only_binary():
    out = os.popen(f"cuobjdump --list-elf {_lib.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out, out


def _u32_step(states, steps):
    s = np.ascontiguousarray(states.copy())
    z = np.zeros(len(s) * steps, np.int64)
    _lib.check(_lib.lib().sfb_host_step_u32(_lib.ptr(s), len(s), steps, _lib.ptr(z)))
    return s, z.reshape(len(s), steps)


def _oracle_steps(states, steps):
    s = states.copy()
    z = np.zeros((len(s), steps), np.int64)
    for w in range(len(s)):
        row = np.ascontiguousarray(s[w])
        for t in range(steps):
            z[w, t] = orc.step(row)
        s[w] = row
    return s, z


def test_u32_step_matches_int64_reference_step():
    rng = np.random.default_rng(1)
    n = 400
    st = np.empty((n, 6), np.int64)
    st[:, :3] = rng.integers(0, sf.M1, size=(n, 3))
    st[:, 3:] = rng.integers(0, sf.M2, size=(n, 3))
    # extreme states: all components at the top of their range, zeros, ones
    st[0] = [sf.M1 - 1] * 3 + [sf.M2 - 1] * 3
    st[1] = [0, 0, 1, 0, 0, 1]
    st[2] = [1, 0, 0, 1, 0, 0]
    st[3] = [sf.M1 - 1, 0, sf.M1 - 1, sf.M2 - 1, 0, sf.M2 - 1]
    st[4] = [2 ** 30, 2 ** 30 - 1, 2 ** 31 - 2, 2 ** 30, 2 ** 31 - 21070, 2 ** 16]
    a, za = _u32_step(st, 300)
    b, zb = _oracle_steps(st, 300)
    assert np.array_equal(za, zb)
    assert np.array_equal(a, b)


def _libm_exp():
    libm = ctypes.CDLL(ctypes.util.find_library("m"))
    libm.exp.argtypes = [ctypes.c_double]
    libm.exp.restype = ctypes.c_double
    return libm.exp


def _bits(x):
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def test_exp_table_matches_host_libm():
    import importlib.util

    spec = importlib.util.spec_from_file_location(
        "gen_exp_data", os.path.join(ROOT, "paper_2201_06604_b200", "csrc", "gen_exp_data.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    consts, tab = mod.extract()
    inc = open(os.path.join(ROOT, "paper_2201_06604_b200", "csrc", "exp_data.inc")).read()
    words = [int(w, 16) for w in re.findall(r"0x([0-9a-f]{16})ull,", inc)]
    assert words == list(tab)
    for name, c in zip(mod.NAMES, consts):
        m = re.search(rf"SFB_EXP_{name}_BITS 0x([0-9a-f]{{16}})ull", inc)
        assert int(m.group(1), 16) == _bits(c)


def test_exp_port_bit_exact_against_libm():
    libm_exp = _libm_exp()
    port = _lib.lib().sfb_host_exp
    rng = np.random.default_rng(7)
    xs = list(rng.uniform(-5.0, 0.0, 60000))          # the Fisher argument range
    xs += list(rng.uniform(-745.5, 709.9, 30000))     # full finite range incl. specialcase
    xs += list(-np.exp(rng.uniform(-60, 2, 10000)))   # tiny to moderate negatives
    xs += list(rng.uniform(-1100, 1100, 2000))        # overflow / underflow
    xs += [0.0, -0.0, 1e-300, -1e-300, 2.0 ** -54, -(2.0 ** -54), 2.0 ** -55, 511.999,
           -511.999, 512.0, -512.0, 700.0, -700.0, 709.78, 709.79, -708.4, -708.5, -744.0,
           -745.1, -745.2, -746.0, 1024.0, -1024.0, math.inf, -math.inf, math.nan,
           5e-324, -5e-324, 1.0, -1.0]
    bad = [x for x in xs if _bits(port(x)) != _bits(libm_exp(x))
           and not (math.isnan(port(x)) and math.isnan(libm_exp(x)))]
    assert not bad, bad[:10]


def test_log1p_port_bit_exact_against_libm():
    libm = ctypes.CDLL(ctypes.util.find_library("m"))
    libm.log1p.argtypes = [ctypes.c_double]
    libm.log1p.restype = ctypes.c_double
    port = _lib.lib().sfb_host_log1p
    rng = np.random.default_rng(3)
    xs = list(-(rng.integers(1, 2 ** 31, 100000) * 2.0 ** -31))  # the fill's arguments
    xs += list(rng.uniform(-1, 1, 50000)) + list(np.exp(rng.uniform(-700, 700, 20000)))
    xs += list(-np.exp(rng.uniform(-60, 0, 20000)))
    xs += [0.0, -0.0, 1e-300, -1e-300, 2.0 ** -54, -(2.0 ** -54), 2.0 ** -29, -(2.0 ** -29),
           0.41422, -0.2929, -0.29289321881345254, 1.0, -1.0, 2.0 ** 53, 2.0 ** 60, math.inf,
           -math.inf, math.nan, -0.999999, 5e-324, -1.5]
    bad = [x for x in xs if _bits(port(x)) != _bits(libm.log1p(x))
           and not (math.isnan(port(x)) and math.isnan(libm.log1p(x)))]
    assert not bad, bad[:10]


def test_log1p_fill_domain_bit_exact_against_libm():
    """The branch-free log1p of the exponential fill (x = -u, u = z 2^-31) ==
    libm log1p bit for bit wherever it does not flag the input as rare, and the
    rare inputs are exactly glibc's other paths (|x| < 2^-29, hu == 0)."""
    libm = ctypes.CDLL(ctypes.util.find_library("m"))
    libm.log1p.argtypes = [ctypes.c_double]
    libm.log1p.restype = ctypes.c_double
    port = _lib.lib().sfb_host_log1p_fill
    rng = np.random.default_rng(9)
    z = np.concatenate([rng.integers(1, 2 ** 31, 300000), np.arange(1, 4097),
                        2 ** 31 - np.arange(1, 4097),
                        # around the k = 0 / k != 0 switch (u = 0.2929) and powers of 2
                        int(0.29289321881345254 * 2 ** 31) + np.arange(-2000, 2001),
                        np.concatenate([(2 ** 31 - 2 ** e) + np.arange(-300, 301)
                                        for e in range(20, 31)])])
    z = z[(z >= 1) & (z < 2 ** 31)]
    flag = ctypes.c_int()
    nrare = 0
    for zi in z:
        x = -(float(zi) * 2.0 ** -31)
        v = port(x, ctypes.byref(flag))
        if flag.value:
            nrare += 1
            continue
        assert _bits(v) == _bits(libm.log1p(x)), (int(zi), v, libm.log1p(x))
    assert nrare < 0.02 * len(z)


def test_printed_matrix_and_goldens(G):
    s4 = sf.create_streams(sf.set_base_creator(), 4)[0]
    assert np.array_equal(s4.matrix(), PRINTED_STREAM_MATRIX)
    st, c = sf.create_streams(sf.set_base_creator(), 1 << 20)
    assert sha(st.current) == G["create_2p20"]["sha"]
    assert list(c.next_seed) == G["create_2p20"]["next_seed"]
    st, c = sf.create_streams(sf.set_base_creator((11, 22, 33, 44, 55, 66)), 300)
    assert sha(st.current) == G["create_toy_300"]["sha"]
    assert np.array_equal(st.current, st.initial)


@pytest.mark.parametrize("e", [0, 1, 10, 134])
def test_jump_matrices(G, e):
    j1, j2 = sf.core._jump_matrices(e)
    assert [list(r) for r in j1] == G[f"jump_{e}"]["j1"]
    assert [list(r) for r in j2] == G[f"jump_{e}"]["j2"]


def test_next_state_and_jumps(G):
    s = sf.StreamState.from_seed(sf.DEFAULT_SEED)
    outs = []
    s0 = s
    for _ in range(2000):
        s, z = sf.next_state(s)
        outs.append(z)
    assert sha(np.array(outs, np.int64)) == G["next_state_2000"]["outs_sha"]
    assert list(s.g1 + s.g2) == G["next_state_2000"]["final"]
    assert s.initial_g1 == (12345,) * 3
    j = sf.jump_ahead(s0, 134)
    assert j.g1 == (336690377, 597094797, 1245771585)
    assert j.g2 == (85196284, 523477687, 2094976052)
    t = sf.StreamState.from_seed((11, 22, 33, 44, 55, 66))
    for e in range(12):
        stepped = t
        for _ in range(2 ** e):
            stepped, _ = sf.next_state(stepped)
        assert sf.jump_ahead(t, e).g1 == stepped.g1
        assert sf.skip_ahead(t, 2 ** e).g2 == stepped.g2
    with pytest.raises(InvalidArgumentError):
        sf.jump_ahead(s0, -1)


def test_creator_validation():
    assert sf.set_base_creator().next_seed == (12345,) * 6
    for bad in [(0, 0, 0, 1, 1, 1), (sf.M1, 1, 1, 1, 1, 1), (1, 1, 1, sf.M2, 1, 1),
                (-1, 1, 1, 1, 1, 1), (1, 2, 3)]:
        with pytest.raises(InvalidSeedError):
            sf.set_base_creator(bad)
    with pytest.raises(InvalidArgumentError):
        sf.create_streams(sf.set_base_creator(), 0)
    a, c = sf.create_streams(sf.set_base_creator(), 2)
    b, _ = sf.create_streams(c, 2)
    full, _ = sf.create_streams(sf.set_base_creator(), 4)
    assert np.array_equal(np.vstack([a.current, b.current]), full.current)


def test_stream_file_format(G, tmp_path):
    s3 = sf.create_streams(sf.set_base_creator(), 3)[0]
    buf = io.StringIO()
    sf.save_streams(s3, buf)
    assert buf.getvalue() == G["save_3"]
    back = sf.load_streams(io.StringIO(buf.getvalue()))
    assert back == s3
    p = tmp_path / "s.txt"
    sf.save_streams(s3, str(p))
    assert p.read_text() == G["save_3"]
    sf.save_streams_atomic(s3, p)
    assert p.read_text() == G["save_3"]
    assert not os.path.exists(str(p) + ".tmp")
    assert sf.load_streams(str(p)) == s3
    # negative / arbitrary int64 values are formatted like Python str(int)
    arr = np.array([[1, -2, 3, 4, 5, 6]], np.int64)
    odd = sf.StreamSet(arr, arr.copy())
    buf = io.StringIO()
    sf.save_streams(odd, buf)
    assert buf.getvalue().splitlines()[1] == "1 -2 3 4 5 6 1 -2 3 4 5 6"


@pytest.mark.parametrize("content", [
    "",
    "wrong-magic v1 count=1\n" + " ".join(["1"] * 12),
    "streamforge-streams v2 count=1\n" + " ".join(["1"] * 12),
    "streamforge-streams v1 count=2\n" + " ".join(["1"] * 12) + "\n",
    "streamforge-streams v1 count=1\n1 2 3\n",
    "streamforge-streams v1 count=1\n" + " ".join(["x"] * 12) + "\n",
    "streamforge-streams v1 count=0\n",
    "streamforge-streams v1 count=x\n",
    "streamforge-streams v1 count=1\n" + " ".join(["1"] * 12) + "\nextra\n",
    "streamforge-streams v1 count=1\n" + " ".join(["0"] * 12) + "\n",
    "streamforge-streams v1 count=1\n" + " ".join([str(sf.M1)] + ["1"] * 11) + "\n",
])
def test_malformed_files_rejected(content):
    with pytest.raises(CorruptStreamFileError):
        sf.load_streams(io.StringIO(content))


def test_parser_accepts_python_int_forms():
    text = ("streamforge-streams v1 count=+1\n"
            "1 0_2 +3 4 5 6 1 2 3 4 5 6\n\n")
    s = sf.load_streams(io.StringIO(text))
    assert s.current.tolist() == [[1, 2, 3, 4, 5, 6]]


def test_round_trip_property():
    rng = np.random.default_rng(3)
    for n in (1, 5, 17):
        cur = np.empty((n, 6), np.int64)
        cur[:, :3] = rng.integers(1, sf.M1, (n, 3))
        cur[:, 3:] = rng.integers(1, sf.M2, (n, 3))
        s = sf.StreamSet(cur.copy(), cur.copy())
        buf = io.StringIO()
        sf.save_streams(s, buf)
        assert sf.load_streams(io.StringIO(buf.getvalue())) == s


def test_checkpoint_files_at_c5_scale(tmp_path):
    # C5 stream count: 2^20 streams create / save / load round trip (C++)
    st, _ = sf.create_streams(sf.set_base_creator(), 1 << 20)
    p = tmp_path / "c5.txt"
    sf.save_streams_atomic(st, p)
    back = sf.load_streams(p)
    assert back == st


def test_api_validation_without_device():
    with pytest.raises(InvalidGridError):
        sf.WorkGrid(0, 4)
    with pytest.raises(InvalidGridError):
        sf.WorkGrid(2, 3).require_paired_lanes()
    assert sf.MatrixBuffer(2, 3).npad == 3
    with pytest.raises(InvalidArgumentError):
        sf.MatrixBuffer(2, 3, npad=2)
    with pytest.raises(InvalidArgumentError):
        sf.FillRequest(shape=(0, 3)).dims()
    with pytest.raises(InvalidArgumentError):
        sf.FillRequest(shape=(1, 2, 3)).dims()
    with pytest.raises(InvalidArgumentError):
        sf.FillRequest(shape=4, kind="poisson").dims()
    with pytest.raises(InvalidRateError):
        sf.FillRequest(shape=4, kind="exponential", rate=0.0).dims()
    assert sf.FillRequest(shape=7).dims() == (1, 7, True)
    assert sf.FillRequest(shape=(7,)).dims() == (1, 7, True)
    streams = sf.create_streams(sf.set_base_creator(), 3)[0]
    with pytest.raises(InsufficientStreamsError):
        sf.run_grid(streams, sf.WorkGrid(2, 2), 2, 2, "uniform")
    with pytest.raises(InvalidGridError):
        sf.fill_normal(sf.create_streams(sf.set_base_creator(), 6)[0],
                       sf.FillRequest(shape=(2, 2), grid=sf.WorkGrid(2, 3)))
    with pytest.raises(InvalidArgumentError):
        sf.ContingencyTable([[5]])
    with pytest.raises(InvalidArgumentError):
        sf.ContingencyTable([[1, -1], [0, 2]])
    with pytest.raises(InvalidMarginsError):
        sf.rcont2([3, 3], [2, 2], np.array([12345] * 6, np.int64))
    month = np.ones((3, 3), np.int64)
    with pytest.raises(InvalidArgumentError):
        sf.fisher_sim(month, 0, sf.create_streams(sf.set_base_creator(), 16)[0],
                      grid=sf.WorkGrid(4, 4))
    with pytest.raises(InsufficientStreamsError):
        sf.fisher_sim(month, 100, sf.create_streams(sf.set_base_creator(), 4)[0],
                      grid=sf.WorkGrid(4, 4))
    g = sf.WorkGrid(256, 64)
    assert sim_num_for(10 ** 6, g) == 1015808
    assert sim_num_for(10 ** 7, g) == 10010624
    assert relaxed_threshold(-47955.0) > -47955.0


def test_thresholds_match_reference(G, A):
    assert sf.logfact_sum(A["month"]) == G["threshold_month"]
    assert sf.logfact_sum(A["week"]) == G["threshold_week"]
    assert sf.logfact_sum(np.array(G["T10"])) == G["threshold_T10"]
    assert np.array_equal(log_factorial_table(int(A["month"].sum())), A["lf_month"])
    t = ContingencyTable(A["month"])
    assert t.row_margins.sum() == t.total == t.col_margins.sum()


def test_element_plan_and_stream_index():
    plan = sf.element_plan(sf.WorkGrid(2, 2), 3, 3)
    assert plan[(0, 0)] == [(0, 0), (0, 2), (2, 0), (2, 2)]
    grid = sf.WorkGrid(2, 2)
    assert sf.stream_index("uniform", grid, 0, 1) == 2
    assert sf.stream_index("normal", grid, 1, 0) == 2
    with pytest.raises(InvalidArgumentError):
        sf.stream_index("uniform", grid, 2, 0)


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU failure mode")
def test_product_path_fails_loudly_without_gpu():
    streams = sf.create_streams(sf.set_base_creator(), 4)[0]
    with pytest.raises(DeviceError):
        sf.fill_uniform(streams, sf.FillRequest(shape=8, grid=sf.WorkGrid(2, 2)))
    with pytest.raises(DeviceError):
        sf.fisher_sim([[1, 2], [3, 4]], 10, streams, grid=sf.WorkGrid(2, 2))


def _host_bm(z1, z2):
    z1 = np.ascontiguousarray(z1, np.int64)
    z2 = np.ascontiguousarray(z2, np.int64)
    a = np.empty(len(z1))
    b = np.empty(len(z1))
    _lib.check(_lib.lib().sfb_host_box_muller(_lib.ptr(z1), _lib.ptr(z2), len(z1),
                                              _lib.ptr(a, _lib._f64p), _lib.ptr(b, _lib._f64p)))
    return a, b


def _bm_draws(n, seed=11):
    rng = np.random.default_rng(seed)
    z1 = rng.integers(1, sf.M1 + 1, n)
    z2 = rng.integers(1, sf.M1 + 1, n)
    # edges: u1 -> 0 and -> 1, powers of two, theta at/near multiples of pi/2
    e1 = [1, 2, 3, 2 ** 30, 2 ** 30 + 1, 2 ** 31 - 2 ** 24, sf.M1 - 1, sf.M1]
    e2 = [1, 2, 2 ** 29 - 1, 2 ** 29, 2 ** 29 + 1, 2 ** 30 - 1, 2 ** 30, 2 ** 30 + 1,
          3 * 2 ** 29 - 1, 3 * 2 ** 29, 3 * 2 ** 29 + 1, 2 ** 28, 2 ** 28 + 1, sf.M1 - 1, sf.M1,
          2 ** 31 - 2 ** 28, 2 ** 31 - 2 ** 28 + 1]
    z1 = np.concatenate([z1, np.repeat(e1, len(e2)), rng.integers(sf.M1 - 2 ** 20, sf.M1 + 1,
                                                                   n // 8)])
    z2 = np.concatenate([z2, np.tile(e2, len(e1)), rng.integers(1, sf.M1 + 1, n // 8)])
    near = np.concatenate([k * 2 ** 29 + np.arange(-50, 51) for k in (1, 2, 3, 4)])
    near = near[(near >= 1) & (near <= sf.M1)]
    z1 = np.concatenate([z1, rng.integers(1, sf.M1 + 1, len(near))])
    z2 = np.concatenate([z2, near])
    return z1, z2


def test_box_muller_port_against_libm():
    """The device Box-Muller (box_muller.cuh), run on the host, against the
    reference formula on glibc (oracle).  Contract:
      f64: |port - ref| <= 4 ulp(ref) or <= 2^-60 absolute;
      f32: |f32(port) - f32(ref)| <= 1 ulp_f32, equal on >= 99.999 %."""
    z1, z2 = _bm_draws(2_000_000)
    a, b = _host_bm(z1, z2)
    ra, rb = orc.box_muller(z1, z2)
    for got, ref in ((a, ra), (b, rb)):
        err = np.abs(got - ref)
        ok = (err <= 4 * np.spacing(np.abs(ref))) | (err <= 2.0 ** -60)
        assert ok.all(), (got[~ok][:4], ref[~ok][:4], z1[~ok][:4], z2[~ok][:4])
        g32, r32 = got.astype(np.float32), ref.astype(np.float32)
        eq = g32 == r32
        d = np.abs(g32.astype(np.float64) - r32.astype(np.float64))
        assert (d <= np.spacing(np.abs(r32)).astype(np.float64)).all()
        assert eq.mean() >= 0.99999, eq.mean()


def _host_bm_f32(z1, z2, newton, seed_err):
    z1 = np.ascontiguousarray(z1, np.int64)
    z2 = np.ascontiguousarray(z2, np.int64)
    a = np.empty(len(z1), np.float32)
    b = np.empty(len(z1), np.float32)
    _lib.check(_lib.lib().sfb_host_box_muller_f32(
        _lib.ptr(z1), _lib.ptr(z2), len(z1), newton, seed_err, _lib.ptr(a, _lib._f32p),
        _lib.ptr(b, _lib._f32p)))
    return a, b


# the device's rsqrt.approx.f64 seed error bound assumed here is asserted on
# the B200 by tests/test_gpu_parity.py::test_rsqrt_seed_accuracy
RSQRT_SEED_BOUND = 2.0 ** -19  # measured on B200: 2^-20.06


@pytest.mark.parametrize("seed_err", [RSQRT_SEED_BOUND, -RSQRT_SEED_BOUND, 0.0])
def test_box_muller_f32_form_against_libm(seed_err):
    """The float32 Box-Muller form (box_muller_pair_f32, the default for
    float32 output), run on the host with a worst-case modelled rsqrt seed,
    against float32(reference formula on glibc).  Contract:
    <= 1 ulp_f32 everywhere (zero crossings included) and identical on
    >= 99.999 % of cells."""
    z1, z2 = _bm_draws(2_000_000)
    a, b = _host_bm_f32(z1, z2, 2, seed_err)  # NEWTON = kBmF32Newton (fill.cu)
    ra, rb = orc.box_muller(z1, z2)
    for got, ref in ((a, ra), (b, rb)):
        r32 = ref.astype(np.float32)
        d = np.abs(got.astype(np.float64) - r32.astype(np.float64))
        ulp = np.spacing(np.abs(r32)).astype(np.float64)
        assert (d <= ulp).all(), (got[d > ulp][:4], r32[d > ulp][:4])
        assert (got == r32).mean() >= 0.99999, (got == r32).mean()


def test_box_muller_f32_form_zero_crossings():
    """theta on and next to fl(k pi/2): both lanes equal float32(reference)."""
    near = np.concatenate([k * 2 ** 29 + np.arange(-5000, 5001) for k in (0, 1, 2, 3, 4)])
    near = near[(near >= 1) & (near <= sf.M1)]
    rng = np.random.default_rng(5)
    z1 = rng.integers(1, sf.M1 + 1, len(near))
    a, b = _host_bm_f32(z1, near, 2, RSQRT_SEED_BOUND)
    ra, rb = orc.box_muller(z1, near)
    for got, ref in ((a, ra), (b, rb)):
        r32 = ref.astype(np.float32)
        d = np.abs(got.astype(np.float64) - r32.astype(np.float64))
        assert (d <= np.spacing(np.abs(r32)).astype(np.float64)).all()


def _host_fisher(table, n, n_items, reps_override=None, stats=False):
    from scipy.special import gammaln

    t = np.asarray(table, np.int64)
    lf = gammaln(np.arange(t.sum() + 1, dtype=np.float64) + 1.0)
    thr = float(-gammaln(t + 1.0).sum())
    thr = thr + 1e-7 * abs(thr)
    reps = reps_override or -(-n // n_items)
    rows, _ = orc.create_streams(sf.DEFAULT_SEED, n_items)
    cur = rows.copy()
    out = np.empty(n_items * reps) if stats else None
    cnt = np.zeros(1, np.int64)
    rm, cm = np.ascontiguousarray(t.sum(1)), np.ascontiguousarray(t.sum(0))
    _lib.check(_lib.lib().sfb_host_fisher_replicates(
        _lib.ptr(cur), _lib.ptr(rm), len(rm), _lib.ptr(cm), len(cm), _lib.ptr(lf, _lib._f64p),
        thr, reps, 0, n_items, None if out is None else _lib.ptr(out, _lib._f64p),
        _lib.ptr(cnt)))
    ref = rows.copy()
    rstats = np.empty(n_items * reps) if stats else None
    rcnt = orc.fisher_replicates(ref, rm, cm, lf, thr, reps, n_items, rstats)
    return int(cnt[0]), rcnt, cur, ref, out, rstats


@pytest.mark.parametrize("name", ["T10", "month", "T4", "week"])
def test_device_fisher_sampler_on_host_matches_oracle(G, A, name):
    """The device sampler source (fisher_sampler.cuh: Markstein walk, exact
    double counters, glibc exp port) run on the host == oracle, bit for bit."""
    table = {"T10": G["T10"], "T4": G["T4"], "month": A["month"], "week": A["week"]}[name]
    cnt, rcnt, cur, ref, st, rst = _host_fisher(table, 0, 64, reps_override=40, stats=True)
    assert cnt == rcnt
    assert np.array_equal(cur, ref)
    assert np.array_equal(st, rst)


@pytest.mark.parametrize("pts,words", [(17, 26), (21, 30)])
def test_device_fisher_sampler_large_memo_budget(G, monkeypatch, pts, words):
    """The background-upgrade memo budgets of the device path -- level 1:
    2^17 points per interior box, 2^26 record words; level 2: 2^21 / 2^30 --
    on T10 (boxes for the large interior cells, long truncated records): the
    sampler run on the host == oracle, bit for bit."""
    monkeypatch.setenv("SFB_MEMO_CELL_PTS_LOG2", str(pts))
    monkeypatch.setenv("SFB_MEMO_WORDS_LOG2", str(words))
    cnt, rcnt, cur, ref, st, rst = _host_fisher(G["T10"], 0, 32, reps_override=40, stats=True)
    assert cnt == rcnt
    assert np.array_equal(cur, ref)
    assert np.array_equal(st, rst)


@pytest.mark.parametrize("key", ["F_E2x2", "F_E2x5", "F_E5x2", "F_Ezero_col", "F_Eones", "F_Ebig"])
def test_device_fisher_sampler_edge_tables(A, key):
    t = A["tab_" + key[2:]]
    cnt, rcnt, cur, ref, st, rst = _host_fisher(t, 0, 16, reps_override=200, stats=True)
    assert cnt == rcnt and np.array_equal(cur, ref) and np.array_equal(st, rst)


def test_device_fisher_sampler_large_margins():
    # margins ~1e6: memo tables hit their budgets / skip rules; results exact
    import time

    t = np.array([[300000, 200000, 150000], [250000, 250000, 1000], [7, 70000, 30000]])
    t0 = time.time()
    cnt, rcnt, cur, ref, st, rst = _host_fisher(t, 0, 8, reps_override=3, stats=True)
    assert time.time() - t0 < 60
    assert cnt == rcnt and np.array_equal(cur, ref) and np.array_equal(st, rst)


def test_status_codes_match_header():
    """Every SFB_E_* code in include/sfb.h maps to the exception class its
    comment names (errors.from_status is the only C-ABI -> Python mapping)."""
    from paper_2201_06604_b200 import errors

    hdr = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                            "include", "sfb.h")).read()
    rows = re.findall(r"#define SFB_E_(\w+) \((-\d+)\)\s+/\* (.*?) \*/", hdr)
    assert len(rows) == 10
    for name, code, comment in rows:
        exc = errors.from_status(int(code), name)
        if name == "IO":
            assert type(exc) is OSError
        elif name == "CUDA":
            assert type(exc) is errors.DeviceError
        else:
            assert type(exc).__name__ in comment, (name, type(exc))
            assert isinstance(exc, errors.StreamforgeError) and exc.status == int(code)
    assert type(errors.from_status(-12345, "x")) is errors.DeviceError


def test_fill_dtype_validation_before_any_launch():
    """run_grid_sharded validates kind/dtype like run_grid
    (grid.py:112-123 order, then the dtype of the kind), and the C-ABI seam
    refuses a buffer whose element size the kernel would overrun."""
    import torch

    from paper_2201_06604_b200.grid import launch_fill
    from paper_2201_06604_b200.sharding import run_grid_sharded

    st = sf.create_streams(sf.set_base_creator(), 16)[0]
    g = sf.WorkGrid(4, 4)
    for kind, dt in [("uniform", np.float32), ("exponential", np.float32),
                     ("uniform-integer", np.float64), ("normal", np.int64),
                     ("uniform", np.int64)]:
        with pytest.raises(InvalidArgumentError):
            run_grid_sharded(st, g, 8, 8, kind, dtype=dt, executor=object())
        with pytest.raises(InvalidArgumentError):
            sf.run_grid(st, g, 8, 8, kind, dtype=dt)
    with pytest.raises(InvalidArgumentError):
        run_grid_sharded(st, g, 8, 8, "poisson", executor=object())
    cur = torch.zeros((16, 6), dtype=torch.int64)
    for kind, tdt in [("uniform", torch.float32), ("exponential", torch.float32),
                      ("uniform-integer", torch.float64), ("normal", torch.int64)]:
        with pytest.raises(InvalidArgumentError):
            launch_fill(kind, cur, 16, torch.empty((8, 8), dtype=tdt), 8, 8, 8, 4, 4)
