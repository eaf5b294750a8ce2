"""`stripley_gpu run` end to end on the device: the
reference's proj/data/sample_result.json reproduced from its own inputs, and
proj/tests/test_cli.cpp's properties (schema, estimation-only stdout, byte-
identical reruns outside telemetry, CSV matrices, --drop-outside, ISO dates)."""
import json
import os
import subprocess

import numpy as np
import pytest

from conftest import golden, surfaces_close
from paper_1912_04753_b200 import build

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(build.nlohmann_include() is None,
                                 reason="nlohmann/json.hpp not available to build the CLI")]

TOL = 1e-9
REPORT_KEYS = ["params", "grid", "k_hat", "l_hat", "theoretical_k", "envelope", "diff_upper",
               "telemetry"]  # proj/data/sample_result.json, in order
PARAM_KEYS = ["points", "boundary", "time_unit", "smax", "tmax", "sims", "sim_method", "seed",
              "index", "cache", "coord_tol", "dist_tol", "partitioner", "partitions", "workers",
              "mode"]


@pytest.fixture(scope="module")
def cli():
    build.build_library()
    path = build.build_cli()
    assert path and os.path.exists(path)
    return path


def run(cli, *args):
    p = subprocess.run([cli, *map(str, args)], capture_output=True, text=True, timeout=600)
    return p.returncode, p.stdout, p.stderr


@pytest.fixture(scope="module")
def sample(tmp_path_factory):
    """proj/data/sample_points.csv + sample_boundary.wkt rebuilt from the golden
    fixture (repr() round-trips every double through std::stod)."""
    g = golden("sample_result.npz")
    d = tmp_path_factory.mktemp("sample")
    pts = d / "sample_points.csv"
    with open(pts, "w") as f:
        f.write("id,x,y,t\n")
        for i, (x, y, t) in enumerate(zip(g["x"], g["y"], g["t"])):
            f.write(f"e{i},{float(x)!r},{float(y)!r},{int(t)}\n")
    wkt = d / "sample_boundary.wkt"
    wkt.write_text("POLYGON((0 0, 10000 0, 10000 10000, 0 10000, 0 0))\n")
    return g, pts, wkt, d


def sample_args(pts, wkt):
    # the flags behind sample_result.json's "params" block
    return ["run", "--points", pts, "--boundary", wkt, "--time-unit", "days", "--smax", 2000,
            "--sstep", 100, "--tmax", 100, "--tstep", 5, "--sims", 19, "--sim-method", "csr",
            "--seed", 42, "--index", "on", "--cache", "on", "--period-start", 0,
            "--period-end", 365]


def test_sample_result_reproduced(cli, sample):
    g, pts, wkt, d = sample
    out = d / "result.json"
    code, _, err = run(cli, *sample_args(pts, wkt), "--out", out)
    assert code == 0, err
    text = out.read_text()
    doc = json.loads(text)
    assert list(doc) == REPORT_KEYS and list(doc["params"]) == PARAM_KEYS
    p = doc["params"]
    assert (p["smax"], p["tmax"], p["sims"], p["seed"], p["sim_method"], p["index"], p["cache"],
            p["mode"], p["partitions"], p["workers"]) == (2000.0, 100, 19, 42, "csr", "on", "on",
                                                          "local", 1, 1)
    assert '"smax": 2000.0,' in text and text.endswith("}\n")  # nlohmann dump(2) formatting
    assert doc["grid"]["s"] == [100.0 * k for k in range(1, 21)]
    assert doc["grid"]["t"] == list(range(5, 101, 5))
    for key, want in [("k_hat", g["k"]), ("l_hat", g["l"]), ("diff_upper", g["diff"])]:
        assert surfaces_close(np.array(doc[key]), want, TOL), key
    assert surfaces_close(np.array(doc["envelope"]["upper_l"]), g["upper"], TOL)
    assert surfaces_close(np.array(doc["envelope"]["lower_l"]), g["lower"], TOL)
    tel = doc["telemetry"]
    assert tel["comparisons"]["in_threshold_pairs"] == int(g["in_threshold_total"])
    assert list(tel) == ["timings", "comparisons", "cache", "redundancy", "bytes", "device"]


def test_reruns_byte_identical_outside_telemetry(cli, sample):
    _, pts, wkt, d = sample
    a, b = d / "a.json", d / "b.json"
    args = ["run", "--points", pts, "--boundary", wkt, "--smax", 300, "--sstep", 100, "--tmax",
            40, "--tstep", 20, "--seed", 5, "--sims", 2, "--sim-method", "csr", "--index", "on",
            "--cache", "on"]
    assert run(cli, *args, "--out", a)[0] == 0
    assert run(cli, *args, "--out", b)[0] == 0
    ja, jb = json.loads(a.read_text()), json.loads(b.read_text())
    ja.pop("telemetry")
    jb.pop("telemetry")
    assert json.dumps(ja) == json.dumps(jb)
    ta, tb = a.read_text(), b.read_text()
    assert ta[:ta.index('"telemetry"')] == tb[:tb.index('"telemetry"')]  # bytes too


def test_schema_permutation_and_estimation_only_stdout(cli, sample):
    _, pts, wkt, d = sample
    base = ["run", "--points", pts, "--boundary", wkt, "--smax", 300, "--sstep", 100, "--tmax",
            40, "--tstep", 20, "--seed", 5, "--period-start", 0, "--period-end", 365]
    out = d / "perm.json"
    code, _, err = run(cli, *base, "--sims", 3, "--sim-method", "permutation", "--out", out)
    assert code == 0, err
    doc = json.loads(out.read_text())
    assert doc["grid"]["s"] == [100.0, 200.0, 300.0] and doc["grid"]["t"] == [20, 40]
    assert len(doc["k_hat"]) == 3 and len(doc["k_hat"][0]) == 2
    assert len(doc["envelope"]["upper_l"]) == 3 and len(doc["diff_upper"]) == 3
    assert doc["params"]["sims"] == 3
    code, stdout, err = run(cli, *base, "--sims", 0)
    assert code == 0, err
    doc = json.loads(stdout)
    assert "k_hat" in doc and "envelope" not in doc and "diff_upper" not in doc


def test_csv_matrices(cli, sample):
    _, pts, wkt, d = sample
    csv_dir = d / "surfaces"
    out = d / "c.json"
    code, _, err = run(cli, "run", "--points", pts, "--boundary", wkt, "--smax", 300, "--sstep",
                       100, "--tmax", 40, "--tstep", 20, "--sims", 2, "--csv-dir", csv_dir,
                       "--out", out)
    assert code == 0, err
    doc = json.loads(out.read_text())
    for name, key in [("k_hat.csv", "k_hat"), ("l_hat.csv", "l_hat"),
                      ("theoretical_k.csv", "theoretical_k"), ("upper_l.csv", None),
                      ("lower_l.csv", None), ("diff_upper.csv", "diff_upper")]:
        path = csv_dir / name
        assert path.exists(), name
        if key:  # 17 significant digits round-trip the JSON's doubles
            m = np.loadtxt(path, delimiter=",", ndmin=2)
            assert np.array_equal(m, np.array(doc[key])), name


def test_drop_outside_and_iso_dates(cli, tmp_path):
    wkt = tmp_path / "b.wkt"
    wkt.write_text("POLYGON((0 0, 1000 0, 1000 1000, 0 1000, 0 0))")
    stray = tmp_path / "stray.csv"
    stray.write_text("id,x,y,t\nin1,100,100,10\nin2,200,300,20\nin3,400,400,30\nout1,5000,100,10\n")
    code, _, err = run(cli, "run", "--points", stray, "--boundary", wkt, "--smax", 300, "--sstep",
                       100, "--tmax", 40, "--tstep", 20, "--sims", 0, "--period-start", 0,
                       "--period-end", 100, "--drop-outside")
    assert code == 0 and "dropped 1 point(s)" in err
    dated = tmp_path / "dated.csv"
    dated.write_text("id,x,y,t\na,100,100,2020-01-01\nb,200,200,2020-01-11\nc,300,300,2020-02-01\n")
    code, stdout, err = run(cli, "run", "--points", dated, "--boundary", wkt, "--time-unit", "days",
                            "--smax", 500, "--sstep", 250, "--tmax", 40, "--tstep", 20,
                            "--sims", 0)
    assert code == 0, err
    assert len(json.loads(stdout)["k_hat"]) == 2


def test_benchmark_matrix(cli, sample):
    _, pts, wkt, _ = sample
    code, stdout, err = run(cli, "run", "--points", pts, "--boundary", wkt, "--smax", 500,
                            "--sstep", 100, "--tmax", 40, "--tstep", 20, "--sims", 4,
                            "--benchmark")
    assert code == 0, err
    rows = [l for l in stdout.splitlines() if l.startswith("index=")]
    assert len(rows) == 8 and len({l.split()[-1] for l in rows}) == 1  # same in-threshold count
