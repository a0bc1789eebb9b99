"""CLI and HTTP front-ends over the B200 backend.

Modelled on the reference's tests/test_cli.py and tests/test_service.py:
exit codes / status codes, output formats and stream-file round trips; every
computed value is checked against the oracle (bit-exact uniforms and Fisher
counts).  Validation paths run on CPU; compute paths are -m gpu.
"""

import numpy as np
import pytest
from click.testing import CliRunner

import paper_2201_06604_b200 as sf
from conftest import PRINTED_STREAM_MATRIX, SIM_1, has_gpu
from oracle import oracle as orc
from paper_2201_06604_b200.command_line import main

import oracle_api as oa


@pytest.fixture
def runner():
    return CliRunner()


def stream_file(path, n=4):
    s, _ = sf.create_streams(sf.set_base_creator(), n)
    sf.save_streams(s, str(path))
    return s


def write_table(path, table):
    path.write_text("\n".join(",".join(str(int(v)) for v in row) for row in table) + "\n")
    return str(path)


def month(A):
    return np.asarray(A["month"], np.int64)


# ----------------------------------------------------------------- CLI, CPU
class TestStreamsCommands:
    def test_create_default_seed_matches_printed_matrix(self, runner, tmp_path):
        out = tmp_path / "s.txt"
        res = runner.invoke(main, ["streams", "create", "--n", "4", "--out", str(out)])
        assert res.exit_code == 0, res.output
        assert np.array_equal(sf.load_streams(str(out)).matrix(), PRINTED_STREAM_MATRIX)

    def test_create_nonpositive_count_exit_2(self, runner, tmp_path):
        res = runner.invoke(main, ["streams", "create", "--n", "0", "--out",
                                   str(tmp_path / "s.txt")])
        assert res.exit_code == 2

    def test_create_refuses_to_clobber(self, runner, tmp_path):
        out = tmp_path / "s.txt"
        out.write_text("keep")
        assert runner.invoke(main, ["streams", "create", "--out", str(out)]).exit_code == 2
        assert out.read_text() == "keep"
        res = runner.invoke(main, ["streams", "create", "--n", "2", "--out", str(out), "--force"])
        assert res.exit_code == 0

    def test_create_bad_seed_exit_2(self, runner, tmp_path):
        for seed in ("1,2,3", "a,b,c,d,e,f", "0,0,0,1,1,1"):
            res = runner.invoke(main, ["streams", "create", "--seed", seed, "--out",
                                       str(tmp_path / "s.txt")])
            assert res.exit_code == 2, seed

    def test_info_prints_matrix(self, runner, tmp_path):
        path = tmp_path / "s.txt"
        stream_file(path)
        res = runner.invoke(main, ["streams", "info", "--file", str(path)])
        assert res.exit_code == 0
        lines = res.output.splitlines()
        assert lines[0] == "4 streams"
        assert np.array_equal(np.array([[int(v) for v in ln.split()] for ln in lines[1:]]),
                              PRINTED_STREAM_MATRIX)

    def test_missing_stream_file_exit_3(self, runner, tmp_path):
        res = runner.invoke(main, ["streams", "info", "--file", str(tmp_path / "none.txt")])
        assert res.exit_code == 3

    def test_corrupt_stream_file_exit_2(self, runner, tmp_path):
        bad = tmp_path / "bad.txt"
        bad.write_text("not a stream file\n")
        assert runner.invoke(main, ["streams", "info", "--file", str(bad)]).exit_code == 2


class TestValidationBeforeCompute:
    def test_generate_needs_exactly_one_of_n_dims(self, runner, tmp_path):
        path = tmp_path / "s.txt"
        stream_file(path)
        args = ["--streams", str(path), "--out", str(tmp_path / "o.csv")]
        assert runner.invoke(main, ["generate"] + args).exit_code == 2
        assert runner.invoke(main, ["generate", "--n", "4", "--dims", "2x2"] + args).exit_code == 2

    def test_generate_bad_grid_text(self, runner, tmp_path):
        path = tmp_path / "s.txt"
        stream_file(path)
        res = runner.invoke(main, ["generate", "--n", "4", "--grid", "2by2", "--streams",
                                   str(path), "--out", str(tmp_path / "o.csv")])
        assert res.exit_code == 2

    def test_normal_odd_lane_grid_exit_2(self, runner, tmp_path):
        path = tmp_path / "s.txt"
        stream_file(path, 6)
        res = runner.invoke(main, ["generate", "--kind", "normal", "--dims", "2x2", "--grid",
                                   "2x3", "--streams", str(path), "--out",
                                   str(tmp_path / "o.csv")])
        assert res.exit_code == 2

    def test_insufficient_streams_exit_2(self, runner, tmp_path):
        path = tmp_path / "s.txt"
        stream_file(path, 2)
        res = runner.invoke(main, ["generate", "--n", "8", "--grid", "2x2", "--streams",
                                   str(path), "--out", str(tmp_path / "o.csv")])
        assert res.exit_code == 2

    def test_fisher_ragged_and_degenerate_tables_exit_2(self, runner, tmp_path):
        path = tmp_path / "s.txt"
        stream_file(path, 16)
        ragged = tmp_path / "r.csv"
        ragged.write_text("1,2,3\n4,5\n")
        one = tmp_path / "one.csv"
        one.write_text("7\n")
        for t in (ragged, one):
            res = runner.invoke(main, ["fisher", "--table", str(t), "--n", "10", "--grid", "4x4",
                                       "--streams", str(path)])
            assert res.exit_code == 2, t

    @pytest.mark.skipif(has_gpu(), reason="checks the no-device exit code")
    def test_no_device_exit_5(self, runner, tmp_path):
        path = tmp_path / "s.txt"
        before = stream_file(path)
        res = runner.invoke(main, ["generate", "--n", "8", "--grid", "2x2", "--streams",
                                   str(path), "--out", str(tmp_path / "o.csv")])
        assert res.exit_code == 5
        assert sf.load_streams(str(path)) == before  # stream file untouched


# ---------------------------------------------------------------- HTTP, CPU
@pytest.fixture(scope="module")
def client():
    from fastapi.testclient import TestClient

    from paper_2201_06604_b200.http_service import app

    return TestClient(app)


def payload(n=4):
    s, _ = sf.create_streams(sf.set_base_creator(), n)
    return {"current": s.current.tolist(), "initial": s.initial.tolist()}


class TestServiceValidation:
    def test_health(self, client):
        r = client.get("/health")
        assert r.status_code == 200 and r.json() == {"status": "ok"}

    def test_streams_create_matches_printed_matrix(self, client):
        r = client.post("/streams/create", json={"n": 4})
        assert r.status_code == 200
        body = r.json()
        got = sf.StreamSet(np.array(body["streams"]["current"], np.int64),
                           np.array(body["streams"]["initial"], np.int64))
        assert np.array_equal(got.matrix(), PRINTED_STREAM_MATRIX)
        _, creator = sf.create_streams(sf.set_base_creator(), 4)
        assert body["next_seed"] == list(creator.next_seed)

    def test_streams_create_422s(self, client):
        assert client.post("/streams/create", json={"n": 0}).status_code == 422
        assert client.post("/streams/create",
                           json={"n": 1, "seed": [0, 0, 0, 1, 1, 1]}).status_code == 422

    def test_generate_422s(self, client):
        assert client.post("/generate", json={"streams": payload(), "n": 4,
                                              "dims": [2, 2]}).status_code == 422
        assert client.post("/generate", json={"streams": payload(2), "n": 8,
                                              "grid": [2, 2]}).status_code == 422
        assert client.post("/generate", json={"streams": payload(), "n": 8,
                                              "kind": "poisson"}).status_code == 422
        assert client.post("/generate", json={"streams": payload(), "n": 8, "grid": [2, 2],
                                              "dtype": "float32"}).status_code == 422

    def test_fisher_invalid_table_422(self, client):
        r = client.post("/fisher", json={"table": [[5]], "n": 10, "streams": payload(16),
                                         "grid": [4, 4]})
        assert r.status_code == 422

    @pytest.mark.skipif(has_gpu(), reason="checks the no-device status code")
    def test_no_device_503(self, client):
        r = client.post("/generate", json={"streams": payload(), "n": 8, "grid": [2, 2]})
        assert r.status_code == 503


# ----------------------------------------------------------------- GPU paths
@pytest.mark.gpu
class TestCliCompute:
    def test_generate_sim1(self, runner, tmp_path):
        path, out = tmp_path / "s.txt", tmp_path / "o.csv"
        stream_file(path)
        res = runner.invoke(main, ["generate", "--n", "8", "--grid", "2x2", "--streams",
                                   str(path), "--out", str(out)])
        assert res.exit_code == 0, res.output
        vals = np.loadtxt(str(out), delimiter=",")
        assert tuple(np.round(vals, 3)) == SIM_1
        ref_st = oa.fresh_states(4)
        ref = oa.fill("uniform", ref_st, 8, (2, 2))
        assert np.array_equal(vals, ref.ravel())  # %.17g round-trips exactly
        assert np.array_equal(sf.load_streams(str(path)).current, ref_st)

    def test_two_runs_continue_one_double_run(self, runner, tmp_path):
        split, full = tmp_path / "a.txt", tmp_path / "b.txt"
        stream_file(split)
        stream_file(full)
        halves = []
        for name in ("h1.csv", "h2.csv"):
            res = runner.invoke(main, ["generate", "--n", "8", "--grid", "2x2", "--streams",
                                       str(split), "--out", str(tmp_path / name)])
            assert res.exit_code == 0
            halves.append(np.loadtxt(str(tmp_path / name), delimiter=","))
        res = runner.invoke(main, ["generate", "--n", "16", "--grid", "2x2", "--streams",
                                   str(full), "--out", str(tmp_path / "f.csv")])
        assert res.exit_code == 0
        assert np.array_equal(np.concatenate(halves),
                              np.loadtxt(str(tmp_path / "f.csv"), delimiter=","))

    @pytest.mark.parametrize("kind", ["uniform", "uniform-integer", "exponential"])
    def test_matrix_kinds_bit_exact_vs_oracle(self, runner, tmp_path, kind):
        path, out = tmp_path / "s.txt", tmp_path / "o.csv"
        stream_file(path, 16)
        res = runner.invoke(main, ["generate", "--kind", kind, "--dims", "20x30", "--grid",
                                   "4x4", "--rate", "0.5", "--streams", str(path), "--out",
                                   str(out)])
        assert res.exit_code == 0, res.output
        got = np.loadtxt(str(out), delimiter=",")
        ref_st = oa.fresh_states(16)
        ref = oa.fill(kind, ref_st, (20, 30), (4, 4), rate=0.5)
        assert np.array_equal(got, ref.astype(np.float64))
        assert np.array_equal(sf.load_streams(str(path)).current, ref_st)

    def test_normal_rerun_byte_identical_any_threads(self, runner, tmp_path):
        outs = []
        for tag, threads in (("1", "1"), ("2", "8")):
            path, out = tmp_path / f"s{tag}.txt", tmp_path / f"o{tag}.csv"
            stream_file(path, 16)
            res = runner.invoke(main, ["generate", "--kind", "normal", "--dims", "20x20",
                                       "--grid", "4x4", "--streams", str(path), "--out",
                                       str(out), "--threads", threads])
            assert res.exit_code == 0
            outs.append(out.read_bytes())
        assert outs[0] == outs[1]

    def test_fisher_month_counts_vs_oracle(self, runner, tmp_path, A):
        path = tmp_path / "s.txt"
        stream_file(path, 16)
        stats_out = tmp_path / "stats.csv"
        t = month(A)
        res = runner.invoke(main, ["fisher", "--table", write_table(tmp_path / "m.csv", t),
                                   "--n", "2000", "--grid", "4x4", "--streams", str(path),
                                   "--stats-out", str(stats_out)])
        assert res.exit_code == 0, res.output
        kv = dict(line.split("=", 1) for line in res.output.splitlines())
        assert round(float(kv["threshold"])) == -47955
        assert int(kv["simNum"]) == 2000
        ref_st = oa.fresh_states(16)
        rstats = np.empty(2000)
        rc = orc.fisher_replicates(ref_st, t.sum(1), t.sum(0), oa.lf_table(int(t.sum())),
                                   oa.relaxed(oa.logfact_sum(t)), 2000 // 16, 16, rstats)
        assert int(kv["counts"]) == rc
        assert float(kv["p.value"]) == (1 + rc) / 2001
        assert np.array_equal(np.loadtxt(str(stats_out), delimiter=","), rstats)
        assert np.array_equal(sf.load_streams(str(path)).current, ref_st)


@pytest.mark.gpu
class TestServiceCompute:
    def test_generate_sim1_and_resume(self, client):
        first = client.post("/generate", json={"streams": payload(), "n": 8,
                                               "grid": [2, 2]}).json()
        assert first["is_vector"] is True
        assert tuple(np.round(np.array(first["values"]).ravel()[:8], 3)) == SIM_1
        second = client.post("/generate", json={"streams": first["streams"], "n": 8,
                                                "grid": [2, 2]}).json()
        full = client.post("/generate", json={"streams": payload(), "n": 16,
                                              "grid": [2, 2]}).json()
        got = np.array(first["values"]).ravel()[:8].tolist() + \
            np.array(second["values"]).ravel()[:8].tolist()
        assert got == np.array(full["values"]).ravel()[:16].tolist()

    def test_float32_normals(self, client):
        r = client.post("/generate", json={"streams": payload(16), "dims": [8, 8],
                                           "grid": [4, 4], "kind": "normal",
                                           "dtype": "float32"})
        assert r.status_code == 200
        got = np.array(r.json()["values"], np.float64)
        ref = oa.fill("normal", oa.fresh_states(16), (8, 8), (4, 4))
        assert np.array_equal(got.astype(np.float32), ref.astype(np.float32))

    def test_fisher_matches_api_and_oracle(self, client, A):
        t = month(A)
        r = client.post("/fisher", json={"table": t.tolist(), "n": 64, "streams": payload(16),
                                         "grid": [4, 4], "return_statistics": True})
        assert r.status_code == 200
        body = r.json()
        expect = sf.fisher_sim(t, 64, sf.create_streams(sf.set_base_creator(), 16)[0],
                               grid=sf.WorkGrid(4, 4), return_stats=True)
        assert body["sim_num"] == expect.sim_num
        assert body["counts"] == expect.counts
        assert body["p_value"] == expect.p_value
        assert body["statistics"] == expect.statistics.tolist()
        assert round(body["threshold"]) == -47955


# ----------------------------------------------------------------- GRF front-ends
def params_file(tmp_path, header="shape,range,variance,anisoRatio,anisoAngleRadians",
                rows=("1.0,2.0,1.0,1.0,0.0", "0.5,3.0,2.0,1.0,0.0")):
    p = tmp_path / "params.csv"
    p.write_text(header + "\n" + "\n".join(rows) + "\n")
    return str(p)


def test_grf_missing_parameter_column_named(runner, tmp_path):
    """reference tests/test_cli.py:238-253."""
    path = tmp_path / "s.txt"
    stream_file(path, 16)
    res = runner.invoke(main, ["grf", "--params", params_file(
        tmp_path, header="shape,range,variance,anisoRatio", rows=("1,2,1,1",)),
        "--ncell-x", "2", "--ncell-y", "2", "--cell-size", "1.0", "--grid", "4x4",
        "--streams", str(path), "--out-dir", str(tmp_path / "o")])
    assert res.exit_code == 2
    assert "anisoAngleRadians" in res.output


@pytest.mark.gpu
class TestGrfFrontends:
    def test_cli_writes_fields_and_manifest(self, runner, tmp_path):
        import json

        path = tmp_path / "s.txt"
        stream_file(path, 16)
        out_dir = tmp_path / "fields"
        res = runner.invoke(main, ["grf", "--params", params_file(tmp_path), "--ncell-x", "5",
                                   "--ncell-y", "4", "--cell-size", "1.0", "--realizations", "2",
                                   "--grid", "4x4", "--streams", str(path), "--out-dir",
                                   str(out_dir)])
        assert res.exit_code == 0, res.output
        manifest = json.loads((out_dir / "manifest.json").read_text())
        assert len(manifest) == 4 and manifest[0]["params"]["shape"] == 1.0
        direct = sf.simulate_grf([sf.MaternParams(1.0, 2.0, 1.0), sf.MaternParams(0.5, 3.0, 2.0)],
                                 sf.GridSpec(5, 4, 1.0), 2,
                                 sf.create_streams(sf.set_base_creator(), 16)[0],
                                 sf.WorkGrid(4, 4))
        for e in manifest:
            f = np.loadtxt(str(out_dir / e["file"]), delimiter=",")
            assert f.shape == (4, 5)
            assert np.array_equal(f, direct[e["parameter_row"] - 1, e["realization"] - 1])

    def test_cli_bin_format_round_trips(self, runner, tmp_path):
        import struct

        outs = {}
        for fmt in ("csv", "bin"):
            path = tmp_path / f"s_{fmt}.txt"
            stream_file(path, 16)
            res = runner.invoke(main, ["grf", "--params", params_file(tmp_path), "--ncell-x",
                                       "3", "--ncell-y", "3", "--cell-size", "1.0", "--grid",
                                       "4x4", "--streams", str(path), "--out-dir",
                                       str(tmp_path / fmt), "--format", fmt])
            assert res.exit_code == 0, res.output
            outs[fmt] = tmp_path / fmt
        raw = (outs["bin"] / "field_p1_r1.bin").read_bytes()
        assert struct.unpack("<IIQ", raw[:16]) == (3, 3, 9)
        assert np.array_equal(np.frombuffer(raw[16:], dtype="<f8").reshape(3, 3),
                              np.loadtxt(str(outs["csv"] / "field_p1_r1.csv"), delimiter=","))

    def test_http_grf_matches_api(self, client):
        r = client.post("/grf", json={"params": [[1.0, 2.0, 1.0, 1.0, 0.0]],
                                      "grid": {"ncell_x": 3, "ncell_y": 3, "cell_size": 1.0},
                                      "n_realizations": 2, "streams": payload(16),
                                      "work_grid": [4, 4]})
        assert r.status_code == 200
        fields = np.array(r.json()["fields"])
        direct = sf.simulate_grf([sf.MaternParams(1.0, 2.0, 1.0)], sf.GridSpec(3, 3, 1.0), 2,
                                 sf.create_streams(sf.set_base_creator(), 16)[0],
                                 sf.WorkGrid(4, 4))
        assert fields.shape == (1, 2, 3, 3) and np.array_equal(fields, direct)

    def test_http_grf_invalid_params_422(self, client):
        r = client.post("/grf", json={"params": [[-1.0, 2.0, 1.0, 1.0, 0.0]],
                                      "grid": {"ncell_x": 2, "ncell_y": 2, "cell_size": 1.0},
                                      "streams": payload(4), "work_grid": [2, 2]})
        assert r.status_code == 422


def test_fisher_plan_cache_keeps_validation_order():
    """plan_fisher caches the host preparation per (table, n, grid); a cache
    hit returns the same plan, still checks the stream count, and invalid
    inputs raise the reference's errors in its order (table, n, streams --
    fisher.py:134-139) whether or not a plan is cached."""
    from paper_2201_06604_b200.errors import (InsufficientStreamsError, InvalidArgumentError)
    from paper_2201_06604_b200.fisher import plan_fisher

    t = [[3, 1], [1, 3]]
    g = sf.WorkGrid(4, 2)
    st = sf.StreamSet(np.ones((8, 6), np.int64), np.ones((8, 6), np.int64))
    small = sf.StreamSet(np.ones((4, 6), np.int64), np.ones((4, 6), np.int64))
    p1 = plan_fisher(t, 100, st, g)
    assert plan_fisher(np.array(t), 100, st, g) is p1
    assert plan_fisher(t, 101, st, g) is not p1
    assert p1.sim_num == 104 and p1.reps == 13
    with pytest.raises(InsufficientStreamsError):
        plan_fisher(t, 100, small, g)          # cache hit: streams still checked
    with pytest.raises(InvalidArgumentError):
        plan_fisher(t, 0, small, g)            # n before streams
    with pytest.raises(InvalidArgumentError):
        plan_fisher([[-1, 2], [1, 1]], 0, small, g)  # table first
    with pytest.raises(InvalidArgumentError):
        plan_fisher([[-1, 2], [1, 1]], 100, st, g)   # never cached
