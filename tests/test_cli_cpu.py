"""The `stripley_gpu run` CLI's argument and ingest behaviour (no GPU needed:
every case fails before the device is touched).  Mirrors the reference's
proj/tests/test_cli.cpp cases "usage errors exit 1", "data errors exit 2 with
the offending line" and "points outside the region are fatal unless dropped"
(the fatal half), plus the ingest rules of proj/core/src/io.cpp."""
import os
import subprocess

import pytest

from paper_1912_04753_b200 import build

pytestmark = pytest.mark.skipif(build.nlohmann_include() is None,
                                reason="nlohmann/json.hpp not available to build the CLI")


@pytest.fixture(scope="module")
def cli():
    build.build_library()
    path = build.build_cli()
    assert path and os.path.exists(path)
    return path


def run(cli, *args):
    p = subprocess.run([cli, *map(str, args)], capture_output=True, text=True, timeout=120)
    return p.returncode, p.stdout + p.stderr


@pytest.fixture()
def files(tmp_path):
    boundary = tmp_path / "b.wkt"
    boundary.write_text("POLYGON((0 0, 1000 0, 1000 1000, 0 1000, 0 0))")
    return tmp_path, boundary


def test_usage_errors_exit_1(cli):
    assert run(cli, "run", "--smax", "10")[0] == 1           # required options missing
    assert run(cli)[0] == 1                                  # no subcommand
    assert run(cli, "frobnicate")[0] == 1
    code, out = run(cli, "run", "--points", "a", "--boundary", "b", "--smax", "1", "--sstep", "1",
                    "--tmax", "1", "--tstep", "1", "--time-unit", "fortnights")
    assert code == 1 and "--time-unit" in out
    assert run(cli, "run", "--points", "a", "--boundary", "b", "--smax", "x", "--sstep", "1",
               "--tmax", "1", "--tstep", "1")[0] == 1
    assert run(cli, "--help")[0] == 0


def test_data_errors_exit_2_with_the_offending_line(cli, files):
    d, boundary = files
    bad = d / "bad.csv"
    bad.write_text("id,x,y,t\na,1,2,3\nb,NOPE,2,3\n")
    code, out = run(cli, "run", "--points", bad, "--boundary", boundary, "--smax", 10, "--sstep",
                    10, "--tmax", 1, "--tstep", 1, "--sims", 0)
    assert code == 2 and ":3" in out and "invalid coordinate" in out
    for body, msg in [("", "empty file"), ("id,x,z,t\n", ":1: expected header id,x,y,t"),
                      ("id,x,y,t\n", "no data rows"), ("id,x,y,t\na,1,2\n", ":2: expected 4 columns"),
                      ("id,x,y,t\na,1,2,2020-13-01\n", "invalid ISO date"),
                      ("id,x,y,t\na,1,2,3.5\n", "invalid timestamp"),
                      ("id,x,y,t\na,inf,2,3\n", "coordinate not finite")]:
        bad.write_text(body)
        code, out = run(cli, "run", "--points", bad, "--boundary", boundary, "--smax", 10,
                        "--sstep", 10, "--tmax", 1, "--tstep", 1, "--sims", 0)
        assert code == 2 and msg in out, (body, out)
    code, out = run(cli, "run", "--points", d / "missing.csv", "--boundary", boundary, "--smax",
                    10, "--sstep", 10, "--tmax", 1, "--tstep", 1)
    assert code == 2 and "cannot open" in out


def test_boundary_formats_and_errors(cli, files):
    d, _ = files
    pts = d / "p.csv"
    pts.write_text("id,x,y,t\nin1,100,100,10\nout1,5000,100,10\n")
    common = ["--smax", 300, "--sstep", 100, "--tmax", 40, "--tstep", 20, "--sims", 0,
              "--period-start", 0, "--period-end", 100]
    for text, msg in [("POLYGON((0 0, 1 0, 1 1, 0 0), (0.2 0.2, 0.3 0.2, 0.3 0.3))", "holes"),
                      ("POLYGON((0 0, 1 x, 1 1))", "malformed WKT coordinate"),
                      ("POLYGON((0 0, 1 1, 0 0))", "polygon needs >= 3 vertices"),
                      ("LINESTRING(0 0, 1 1)", "boundary must be WKT POLYGON or GeoJSON Polygon"),
                      ('{"type": "Point", "coordinates": [0, 0]}', "must be a Polygon"),
                      ('{"type": "Polygon", "coordinates": [[[0,0],[1,0],[1,1]], [[0,0]]]}',
                       "holes"),
                      ('{"type": ', "invalid GeoJSON"), ("", "empty boundary file")]:
        b = d / "bnd.txt"
        b.write_text(text)
        code, out = run(cli, "run", "--points", pts, "--boundary", b, *common)
        assert code == 2 and msg in out, (text, out)
    # a valid GeoJSON Feature; out1 is outside -> fatal, listing its id
    b = d / "bnd.geojson"
    b.write_text('{"type": "Feature", "geometry": {"type": "Polygon", "coordinates": '
                 '[[[0,0],[1000,0],[1000,1000],[0,1000],[0,0]]]}}')
    code, out = run(cli, "run", "--points", pts, "--boundary", b, *common)
    assert code == 2 and "out1" in out and "--drop-outside" in out


def test_points_outside_fatal_lists_ids(cli, files):
    d, boundary = files
    stray = d / "stray.csv"
    stray.write_text("id,x,y,t\nin1,100,100,10\nin2,200,300,20\nin3,400,400,30\nout1,5000,100,10\n")
    code, out = run(cli, "run", "--points", stray, "--boundary", boundary, "--smax", 300,
                    "--sstep", 100, "--tmax", 40, "--tstep", 20, "--sims", 0, "--period-start", 0,
                    "--period-end", 100)
    assert code == 2 and "1 point(s) outside study region/period: out1" in out


def test_invalid_grid_is_a_data_error(cli, files):
    d, boundary = files
    pts = d / "p.csv"
    pts.write_text("id,x,y,t\na,100,100,10\nb,200,200,20\n")
    # smax < sstep: an empty grid (estimator.cpp:15-16: "distance grid must be non-empty")
    code, out = run(cli, "run", "--points", pts, "--boundary", boundary, "--smax", 50,
                    "--sstep", 100, "--tmax", 40, "--tstep", 20)
    assert code == 2 and "distance grid must be non-empty" in out, out
