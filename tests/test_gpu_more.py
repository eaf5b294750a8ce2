"""GPU parity, second set: the C++ reference-facing API, null models, edge
cases of the reference's tests, multi-rank combination, larger configs.

Bars as in test_gpu_parity.py: bit-exact counts / points / bins; weighted
K/L within TOL = 1e-9 relative (north_star), typically ~1e-15.
"""
import json
import os
import subprocess
import tempfile

import numpy as np
import pytest

from conftest import ROOT, golden, rel_err, surfaces_close

pytestmark = pytest.mark.gpu
TOL = 1e-9


@pytest.fixture(scope="module")
def api():
    from paper_1912_04753_b200.stripley import device, est, geom, rt, sim

    device.get(0)
    return dict(est=est, geom=geom, rt=rt, sim=sim, dev=device.get(0))


@pytest.fixture(scope="module")
def port():
    from oracle import port

    return port


def square(side, p0=0, p1=100):
    return np.array([[0, 0], [side, 0], [side, side], [0, side]], float), p0, p1


# ------------------------------------------------------------ C++ API
def _write(path, *arrays):
    with open(path, "wb") as f:
        for a in arrays:
            f.write(np.asarray(a).tobytes())


def test_cpp_api_selftest():
    from paper_1912_04753_b200.build import build_cpp_tests

    exe = build_cpp_tests()
    r = subprocess.run([exe, "selftest"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "failures=0" in r.stdout


@pytest.mark.parametrize("world", [1, 2, 3])
def test_cpp_run_job_golden_sample(world):
    """rt::run_job through the C++ API on proj/data/sample_result.json's input;
    world > 1 emulates ranks sequentially through the exact reduction hooks."""
    from paper_1912_04753_b200.build import build_cpp_tests

    exe = build_cpp_tests()
    g = golden("sample_result.npz")
    with tempfile.TemporaryDirectory() as d:
        pts, ring, grid = (os.path.join(d, f) for f in ("p.bin", "r.bin", "g.bin"))
        n = len(g["x"])
        _write(pts, np.uint64(n), g["x"], g["y"], g["t"].astype(np.int64))
        _write(ring, np.uint64(g["ring"].size), g["ring"].reshape(-1))
        _write(grid, np.uint64(len(g["s"])), g["s"], np.uint64(len(g["tv"])), g["tv"].astype(np.int64))
        r = subprocess.run([exe, "runjob", pts, ring, "0", "365", grid, str(int(g["sims"])),
                            str(int(g["seed"])), str(world)], capture_output=True, text=True,
                           timeout=300)
    assert r.returncode == 0, r.stderr
    out = json.loads(r.stdout)
    shape = g["k"].shape
    for key in ("k", "l", "upper", "lower", "diff"):
        assert surfaces_close(np.array(out[key]).reshape(shape), g[key], TOL), key


# ------------------------------------------------------------ null models
def test_device_bootstrap_and_permutation_bit_exact(api, port):
    import ctypes as C

    from paper_1912_04753_b200 import _lib

    dev, geom = api["dev"], api["geom"]
    g = golden("sample_result.npz")
    x, y, t = g["x"], g["y"], g["t"].astype(np.int64)
    dev.configure(geom.StudyRegion(g["ring"], 0, 365))
    n = len(x)
    for method, ref_fn in ((1, port.generate_bootstrap), (2, port.generate_permutation)):
        for seed in (1, 42, 2**40 + 7):
            ox, oy, ot = np.zeros(n), np.zeros(n), np.zeros(n, np.int64)
            dev.check(dev.lib.stk_generate(dev.h, method, n, _lib.ptr(x), _lib.ptr(y),
                                           _lib.ptr(t, C.c_int64), seed, _lib.ptr(ox), _lib.ptr(oy),
                                           _lib.ptr(ot, C.c_int64)))
            rx, ry, rt_ = ref_fn(x, y, t, seed)
            assert np.array_equal(ox, rx) and np.array_equal(oy, ry) and np.array_equal(ot, rt_)


@pytest.mark.parametrize("method", [1, 2])
def test_run_simulations_null_models_vs_port(api, port, method):
    est, geom, sim = api["est"], api["geom"], api["sim"]
    g = golden("sample_result.npz")
    x, y, t, ring = g["x"], g["y"], g["t"], g["ring"]
    region = geom.StudyRegion(ring, 0, 365)
    grid = est.DistanceGrid(g["s"], g["tv"])
    surfs = sim.run_simulations((x, y, t), region, grid, sim.Method(method), 4, 9)
    gen = port.generate_bootstrap if method == 1 else port.generate_permutation
    for r in range(4):
        sx, sy, st = gen(x, y, t, 9 + r)
        want = port.estimate(sx, sy, st, ring, 0, 365, g["s"], g["tv"])["l"]
        assert surfaces_close(surfs[r].values, want, TOL), r


# ------------------------------------------------------------ edge cases
def _compare(api, port, x, y, t, ring, p0, p1, s, tv, tol=TOL):
    est, geom = api["est"], api["geom"]
    region = geom.StudyRegion(ring, p0, p1)
    grid = est.DistanceGrid(s, tv)
    h = est.pair_histogram((x, y, t), region, grid)
    o = port.pair_histogram(x, y, t, ring, p0, p1, np.asarray(s, float), np.asarray(tv, np.int64))
    assert np.array_equal(h["counts"], o["counts"])
    assert rel_err(h["hist"], o["hist"]) <= 1e-13
    k = est.estimate_surface((x, y, t), region, grid)
    ko = port.finalize(o["hist"], len(x), port.area(ring), p1 - p0)
    assert surfaces_close(k.values, ko, tol)
    return h


def test_coincident_points_pair_with_weight_one(api, port):
    """Self-exclusion is by index; coincident distinct points pair at d = 0
    with omega = 1 (edge_correction.cpp:47).  The circle around (50, 50)
    through all four corners gets omega == 0 from the reference's arc rule:
    1/0 = inf enters that bin, whose K is NaN in the reference (checked
    against oracle/_ref when it is built here)."""
    ring, p0, p1 = square(100.0)
    x = np.array([0.0, 0.0, 50.0, 50.0, 50.0, 100.0])
    y = np.array([0.0, 0.0, 50.0, 50.0, 50.0, 100.0])
    t = np.array([0, 0, 10, 10, 12, 100])
    h = _compare(api, port, x, y, t, ring, p0, p1, [1.0, 10.0, 200.0], [1, 5, 100])
    assert h["counts"][0, 0] == 4  # (0,0)x2 at u=0 and the two (50,50) points at u=0
    assert h["counts"][0, 1] == 4  # (50,50) pairs at u=2
    assert np.isnan(h["hist"][2, 2]) and h["counts"][2, 2] == 22
    assert h["sum_hi"][2, 2] >= 1 << 56  # the exported infinite-term mark (stk.h)
    est, geom = api["est"], api["geom"]
    k = est.estimate_surface((x, y, t), geom.StudyRegion(ring, p0, p1),
                             est.DistanceGrid([1.0, 10.0, 200.0], [1, 5, 100]))
    assert np.isnan(k.values[2, 2]) and np.isfinite(k.values[:2]).all()


def test_points_on_boundary_corners_and_period_ends(api, port):
    ring, p0, p1 = square(1000.0, 0, 1000)
    rng = np.random.default_rng(1)
    n = 400
    x = rng.uniform(0, 1000, n)
    y = rng.uniform(0, 1000, n)
    t = rng.integers(0, 1000, n, endpoint=True)
    x[:40] = 0.0          # left edge
    y[40:80] = 1000.0     # top edge
    x[80:90] = 1000.0; y[80:90] = 0.0  # corner
    t[90:120] = 0         # period start
    t[120:150] = 1000     # period end
    _compare(api, port, x, y, t, ring, p0, p1, [50.0, 125.0, 250.0, 400.0], [10, 100, 300])


def test_thresholds_inclusive_exact_distances(api, port):
    """d == s_k and u == t_l land in bin k / l (lower_bound, inclusive)."""
    ring, p0, p1 = square(1000.0, 0, 100)
    x = np.array([100.0, 130.0, 100.0, 100.0, 500.0])
    y = np.array([100.0, 140.0, 150.0, 100.0, 500.0])  # distances 50 (3-4-5), 50, 0
    t = np.array([10, 20, 30, 10, 50])
    h = _compare(api, port, x, y, t, ring, p0, p1, [25.0, 50.0], [10, 20])
    assert h["counts"].sum() > 0


def test_single_cell_all_pairs(api, port):
    """C3-like: s_max and t_max exceed the box, so every pair is in threshold."""
    ring, p0, p1 = square(1000.0, 0, 8_640_000)
    from oracle import port as orc

    x, y, t = orc.generate_cstr(3000, ring, p0, p1, 3)
    s = [93.75 * (k + 1) for k in range(16)]
    tv = [540_000 * (k + 1) for k in range(16)]
    h = _compare(api, port, x, y, t, ring, p0, p1, s, tv)
    assert int(h["counts"].sum()) == 3000 * 2999


def test_dense_arc_pairs_with_duplicates(api, port):
    """Every pair near a corner, many exact duplicates (bootstrap-like): the
    densest arc-path load per warp (stresses the per-warp arc ring)."""
    ring, p0, p1 = square(1000.0, 0, 100)
    rng = np.random.default_rng(7)
    base_x = rng.uniform(0, 60, 200)
    base_y = rng.uniform(0, 60, 200)
    base_t = rng.integers(0, 100, 200, endpoint=True)
    pick = rng.integers(0, 200, 2500)
    x, y, t = base_x[pick], base_y[pick], base_t[pick]
    _compare(api, port, x, y, t, ring, p0, p1, [10.0, 40.0, 90.0], [20, 60, 100])


def test_wide_period_64bit_times(api, port):
    """Study periods >= 2^31 time units take the 64-bit-time kernel."""
    p0, p1 = -(1 << 40), (1 << 40) + 12345
    ring = np.array([[0, 0], [2000, 0], [2000, 2000], [0, 2000]], float)
    rng = np.random.default_rng(11)
    n = 3000
    x = rng.uniform(0, 2000, n)
    y = rng.uniform(0, 2000, n)
    t = rng.integers(p0, p1, n, endpoint=True)
    t[:1500] = rng.integers(-(1 << 33), 1 << 33, 1500)  # dense middle: many temporal pairs
    tv = [1 << 30, 1 << 31, 1 << 33, 1 << 35]
    _compare(api, port, x, y, t, ring, p0, p1, [100.0, 300.0, 600.0], tv)


def test_one_bin_grid_and_tiny_n(api, port):
    ring, p0, p1 = square(10.0, 0, 10)
    _compare(api, port, np.array([1.0, 2.0]), np.array([1.0, 2.0]), np.array([0, 10]), ring, p0,
             p1, [20.0], [20])


def test_star_polygons_bitmask_and_fallback_paths(api, port):
    """14- and 64-vertex rings: the >32-vertex ring takes the general path,
    and circles with > 8 crossings take the fallback."""
    g = golden("weights.npz")
    for k in (1, 3):  # 12-vertex star, 64-vertex star
        ring = g[f"{k}_ring"]
        cx, cy = g[f"{k}_cx"][:300], g[f"{k}_cy"][:300]
        rng = np.random.default_rng(k)
        t = rng.integers(0, 100, len(cx))
        span = float(np.ptp(ring[:, 0]))
        s = [span * f for f in (0.1, 0.3, 0.6, 1.0)]
        _compare(api, port, cx, cy, t, ring, 0, 100, s, [10, 50, 100])


def test_deterministic_across_runs(api):
    est, geom, sim = api["est"], api["geom"], api["sim"]
    ring, p0, p1 = square(5000.0, 0, 1_000_000)
    region = geom.StudyRegion(ring, p0, p1)
    grid = est.DistanceGrid([100.0 * (k + 1) for k in range(10)], [50_000 * (k + 1) for k in range(8)])
    pts = sim.generate_cstr(20_000, region, 5)
    a = est.pair_histogram(pts, region, grid)
    b = est.pair_histogram(pts, region, grid)
    assert np.array_equal(a["sum_hi"], b["sum_hi"]) and np.array_equal(a["sum_lo"], b["sum_lo"])
    k1 = est.estimate_surface(pts, region, grid).values
    k2 = est.estimate_surface(pts, region, grid).values
    assert np.array_equal(k1, k2)


# ------------------------------------------------------------ multi-rank
def test_run_job_ranks_combine_bit_identically(api):
    """rt.run_job's multi-process path (stk_run_job_shard per rank + exact
    SUM / MAX / MIN) emulated sequentially: identical K at any world size."""
    import ctypes as C

    from paper_1912_04753_b200 import _lib

    est, geom, rt = api["est"], api["geom"], api["rt"]
    dev = api["dev"]
    g = golden("sample_result.npz")
    region = geom.StudyRegion(g["ring"], 0, 365)
    grid = est.DistanceGrid(g["s"], g["tv"])
    x, y, t = (np.ascontiguousarray(a) for a in (g["x"], g["y"], g["t"].astype(np.int64)))
    dev.configure(region, grid)
    shape = g["k"].shape
    single = rt.run_job((x, y, t), region, rt.JobSpec(grid=grid, sims=19, seed=42))
    for world in (2, 4):
        cnt = np.zeros(shape, object); tot = np.zeros(shape, object)
        up = np.full(shape, -np.inf); lo = np.full(shape, np.inf)
        for rank in range(world):
            r0, r1 = rt.shard_range(19, rank, world)
            c_ = np.zeros(shape, np.uint64); hi = np.zeros(shape, np.uint64)
            lw = np.zeros(shape, np.uint64)
            u_ = np.full(shape, -np.inf); l_ = np.full(shape, np.inf)
            tel = _lib.StkTelemetry()
            dev.check(dev.lib.stk_run_job_shard(
                dev.h, _lib.ptr(x), _lib.ptr(y), _lib.ptr(t, C.c_int64), len(x), rank, world,
                r0, r1, 42, 0, _lib.ptr(c_, C.c_uint64), _lib.ptr(hi, C.c_uint64),
                _lib.ptr(lw, C.c_uint64), _lib.ptr(u_), _lib.ptr(l_), C.byref(tel)))
            cnt += c_.astype(object)
            tot += hi.astype(object) * (1 << 64) + lw.astype(object)
            up = np.maximum(up, u_); lo = np.minimum(lo, l_)
        hi = np.array([[int(v) >> 64 for v in row] for row in tot], np.uint64)
        lw = np.array([[int(v) & ((1 << 64) - 1) for v in row] for row in tot], np.uint64)
        k, l = est.finalize_exact(hi, lw, len(x), region, grid)
        assert np.array_equal(k.values, single.k_hat.values)
        assert np.array_equal(l.values, single.l_hat.values)
        assert np.array_equal(up, single.upper_l.values)
        assert np.array_equal(lo, single.lower_l.values)
        assert np.array_equal(cnt.astype(np.uint64),
                              est.pair_histogram((x, y, t), region, grid)["counts"])


# ------------------------------------------------------------ larger configs
def test_c2_observed_thomas_full_size(api, port):
    """configs[1]'s observed pattern (N ~ 100k Thomas clusters): counts bit-exact."""
    from paper_1912_04753_b200 import configs

    cfg = configs.CONFIGS["C2"]
    s, tv = configs.grid_values(cfg)
    x, y, t = configs.thomas(cfg)
    _compare(api, port, x, y, t, cfg.ring(), 0, cfg.period_s, s, tv)


@pytest.mark.slow
def test_c3_full_size_properties(api):
    """configs[2] at full N = 200,000 (4e10 pairs): every ordered pair in
    threshold; K monotone; the top cell of K equals A*D/n^2 * sum of 1/w,
    with total count N(N-1)."""
    from paper_1912_04753_b200 import configs

    est, geom, sim = api["est"], api["geom"], api["sim"]
    cfg = configs.CONFIGS["C3"]
    s, tv = configs.grid_values(cfg)
    region = geom.StudyRegion(cfg.ring(), 0, cfg.period_s)
    grid = est.DistanceGrid(s, tv)
    pts = sim.generate_cstr(cfg.n, region, cfg.seed)
    h = est.pair_histogram(pts, region, grid)
    assert int(h["counts"].sum()) == cfg.n * (cfg.n - 1)
    k = est.estimate_surface(pts, region, grid).values
    assert np.all(np.diff(k, axis=0) >= 0) and np.all(np.diff(k, axis=1) >= 0)
    scale = region.area() * region.duration() / float(cfg.n) ** 2
    assert k[-1, -1] == pytest.approx(scale * h["hist"].sum(), rel=1e-12)


def test_bin_tables_close_thresholds_and_wide_range(api, port):
    """The log-scale q buckets and linear u buckets: thresholds closer than a
    bucket (the device falls back to the compare loop), a grid spanning six
    decades, and distances / lags landing exactly on thresholds."""
    ring, p0, p1 = square(1000.0, 0, 10_000)
    rng = np.random.default_rng(77)
    n = 3000
    x = rng.uniform(0, 1000, n)
    y = rng.uniform(0, 1000, n)
    t = rng.integers(0, 10_001, n)
    # exact-threshold pairs: points at integer offsets from a few anchors
    for a in range(10):
        x[a * 3:a * 3 + 3] = [100.0 + 50 * a, 100.0 + 50 * a + 3.0, 100.0 + 50 * a]
        y[a * 3:a * 3 + 3] = [500.0, 504.0, 505.0]
        t[a * 3:a * 3 + 3] = [5000, 5020, 5040]
    close = [5.0, 5.0 + 1e-9, 5.0 + 2e-9, 20.0, 20.000001, 100.0, 250.0]
    _compare(api, port, x, y, t, ring, p0, p1, close, [20, 21, 22, 40, 500])
    wide = [1e-3, 1e-2, 0.1, 1.0, 5.0, 10.0, 100.0, 300.0]
    _compare(api, port, x, y, t, ring, p0, p1, wide, [1, 2, 3, 20, 40, 9000])


def test_evenly_spaced_time_bins(api, port):
    """Evenly spaced time thresholds T_k = T_0 + k D take the multiply-high t
    bin (BinView::t_uni): offsets T_0 below, at and above D (t = 0 is not a valid threshold), D = 2, large D,
    and lags exactly on, one below and one above every threshold."""
    ring, p0, p1 = square(1000.0, 0, 200_000)
    rng = np.random.default_rng(91)
    n = 2500
    x = rng.uniform(0, 1000, n)
    y = rng.uniform(0, 1000, n)
    t = rng.integers(0, 200_001, n)
    s = [10.0, 20.0, 40.0, 80.0]
    for t0, d, ct in [(7, 13, 9), (13, 13, 6), (40, 13, 5), (2, 2, 40), (1, 2, 33),
                      (5000, 9999, 12)]:
        tv = [t0 + k * d for k in range(ct)]
        # lags on, just below and just above each threshold from a few anchors
        xx, yy, tt = x.copy(), y.copy(), t.copy()
        m = 0
        for k, T in enumerate(tv):
            for du in (T - 1, T, T + 1):
                if du < 0 or m + 2 > n:
                    continue
                xx[m:m + 2] = [300.0 + k, 300.0 + k + 1.0]
                yy[m:m + 2] = [600.0 + m, 600.0 + m]
                tt[m:m + 2] = [50_000, 50_000 + du]
                m += 2
        _compare(api, port, xx, yy, tt, ring, p0, p1, s, tv)


def test_dense_cell_item_parts(api, port):
    """A cluster of 5,000 points inside one grid cell (> kPartCells): items
    are walked as several parts by different warps; sums must not change."""
    ring, p0, p1 = square(10_000.0, 0, 1000)
    rng = np.random.default_rng(31)
    a = rng.uniform(0, 2 * np.pi, 5000)
    rad = 18.0 * np.sqrt(rng.uniform(0, 1, 5000))
    x = np.concatenate([5025.0 + rad * np.cos(a), rng.uniform(0, 10_000, 2000)])
    y = np.concatenate([5025.0 + rad * np.sin(a), rng.uniform(0, 10_000, 2000)])
    t = np.concatenate([rng.integers(0, 40, 5000), rng.integers(0, 1001, 2000)])
    h = _compare(api, port, x, y, t, ring, p0, p1, [5.0, 20.0, 50.0, 100.0], [10, 50, 200])
    assert int(h["counts"].sum()) > 20_000_000


def test_utm_offset_clusters_integer_bucket_bins(api, port):
    """UTM-like coordinates (a 20 km rectangle at x0 = 500 km, y0 = 4,000 km)
    with clustered points, a distance grid spanning 10 m .. 2.5 km and a
    lag grid in days: the integer-bit distance buckets (high word of q) and
    power-of-two lag buckets must give the reference's bins bit for bit, and
    points placed exactly on thresholds must land in the inclusive bin."""
    x0, y0 = 500_000.0, 4_000_000.0
    ring = np.array([[x0, y0], [x0 + 20_000, y0], [x0 + 20_000, y0 + 20_000], [x0, y0 + 20_000]])
    p0, p1 = 0, 365 * 86400
    rng = np.random.default_rng(2024)
    cx = rng.uniform(x0 + 500, x0 + 19_500, 40)
    cy = rng.uniform(y0 + 500, y0 + 19_500, 40)
    ct = rng.integers(p0 + 86400, p1 - 86400, 40)
    k = rng.integers(0, 40, 6000)
    x = np.clip(cx[k] + rng.normal(0, 300, 6000), x0, x0 + 20_000)
    y = np.clip(cy[k] + rng.normal(0, 300, 6000), y0, y0 + 20_000)
    t = np.clip(ct[k] + rng.normal(0, 5 * 86400, 6000).astype(np.int64), p0, p1)
    # exact-threshold pairs: offsets of 10, 100 and 2500 m along x, lags of 1 and 30 days
    for j, (dx, du) in enumerate([(10.0, 86400), (100.0, 30 * 86400), (2500.0, 0)]):
        x[2 * j], y[2 * j], t[2 * j] = x0 + 7000.0, y0 + 7000.0 + 50 * j, 100 * 86400
        x[2 * j + 1], y[2 * j + 1], t[2 * j + 1] = x0 + 7000.0 + dx, y0 + 7000.0 + 50 * j, 100 * 86400 + du
    s = [10.0, 25.0, 50.0, 100.0, 250.0, 500.0, 1000.0, 2500.0]
    tv = [86400, 7 * 86400, 30 * 86400, 90 * 86400]
    h = _compare(api, port, x, y, t, ring, p0, p1, s, tv)
    assert int(h["counts"].sum()) > 1_000_000


def test_forced_multi_batch_bit_identical(api):
    """run_pipeline's batch loop (stk_capi.cu): a job forced into >= 3 batches by
    stk_set_memory_budget (the envelope fold across batches, per-batch seed
    offsets of the ladder seed + r, observed pattern only in the first batch)
    equals the single-batch job bit for bit, as do the realisations' L
    surfaces and the in-threshold total (runtime.cpp:207-245)."""
    import ctypes as C

    from paper_1912_04753_b200 import _lib

    est, geom, rt, sim, dev = api["est"], api["geom"], api["rt"], api["sim"], api["dev"]
    ring, p0, p1 = square(5000.0, 0, 200 * 86400)
    region = geom.StudyRegion(ring, p0, p1)
    grid = est.DistanceGrid.regular(50.0, 500.0, 86400, 20 * 86400)
    pts = sim.generate_cstr(20000, region, 99, device=0)
    n, sims, seed = len(pts), 11, 123
    shape = (grid.cells_s(), grid.cells_t())

    def job():
        outs = [np.zeros(shape) for _ in range(5)]
        tel = _lib.StkTelemetry()
        dev.check(dev.lib.stk_run_job(dev.h, _lib.ptr(pts.x), _lib.ptr(pts.y),
                                      _lib.ptr(pts.t, C.c_int64), n, sims, seed, 0,
                                      *[_lib.ptr(o) for o in outs], C.byref(tel)))
        l_all, up, lo = sim.simulate(pts, region, grid, sim.Method.Cstr, 0, sims, seed, True,
                                     device=0)
        return outs, tel, l_all, up, lo

    dev.configure(region, grid)
    one, tel1, l1, u1, d1 = job()
    assert tel1.batches == 1
    try:
        dev.set_memory_budget(6 << 20)  # ~4 patterns of 20k points per batch
        many, teln, ln, un, dn = job()
    finally:
        dev.set_memory_budget(16 << 30)
    assert teln.batches >= 3, teln.batches
    for a, b in zip(one, many):
        assert np.array_equal(a, b)
    assert teln.in_threshold_pairs == tel1.in_threshold_pairs
    assert np.array_equal(l1, ln) and np.array_equal(u1, un) and np.array_equal(d1, dn)
    assert np.array_equal(many[2], ln.max(0)) and np.array_equal(many[3], ln.min(0))


def test_reference_program_compiles_and_runs_unchanged():
    """A program written against the reference's runtime.hpp (LocalExecutor,
    a user Executor plug-in with the three virtuals, run_job, RunTelemetry,
    speedup_factor) built against include/stripley/ reproduces the golden
    sample (proj/data/sample_result.json) through both executors and through
    LocalExecutor::run + aggregate on the device."""
    from paper_1912_04753_b200.build import build_reference_program

    exe = build_reference_program()
    g = golden("sample_result.npz")
    with tempfile.TemporaryDirectory() as d:
        pts, ring, grid = (os.path.join(d, f) for f in ("p.bin", "r.bin", "g.bin"))
        n = len(g["x"])
        _write(pts, np.uint64(n), g["x"], g["y"], g["t"].astype(np.int64))
        _write(ring, np.uint64(g["ring"].size), g["ring"].reshape(-1))
        _write(grid, np.uint64(len(g["s"])), g["s"], np.uint64(len(g["tv"])), g["tv"].astype(np.int64))
        r = subprocess.run([exe, pts, ring, "0", "365", grid, str(int(g["sims"])),
                            str(int(g["seed"]))], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    out = json.loads(r.stdout)
    shape = g["k"].shape
    for key, gk in (("k", "k"), ("l", "l"), ("upper", "upper"), ("lower", "lower"),
                    ("diff", "diff"), ("k_plugin", "k"), ("upper_plugin", "upper")):
        assert surfaces_close(np.array(out[key]).reshape(shape), g[gk], TOL), key
    obs = golden("sample_result.npz")["counts_observed"]
    assert surfaces_close(np.array(out["k_tasks"]).reshape(shape), g["k"], TOL)
    assert out["in_threshold"] == int(g["in_threshold_total"])
    assert out["in_threshold_plugin"] == int(g["in_threshold_total"])
    assert out["partition_count"] == 1
    assert out["cylinder_assignments"] == n * (1 + int(g["sims"]))
    assert out["plugin_bytes_sent"] == 1 + int(g["sims"])  # tasks the plug-in ran
    assert out["plugin_bytes_received"] == 1              # plans broadcast
    assert out["ratio"] == 4.0
    assert int(obs.sum()) > 0


def test_nccl_world1_collective_bit_identical(api):
    """The in-library NCCL path (stk_comm_init + stk_run_job_dist: the exact
    limb SUM and MAX/MIN all-reduces and the device finalize) at world 1 gives
    stk_run_job's results bit for bit; the C++ DeviceExecutor rejects world > 1
    without a communicator or hooks."""
    est, geom, rt = api["est"], api["geom"], api["rt"]
    g = golden("sample_result.npz")
    region = geom.StudyRegion(g["ring"], 0, 365)
    grid = est.DistanceGrid(g["s"], g["tv"])
    pts = (g["x"], g["y"], g["t"])
    spec = rt.JobSpec(grid=grid, sims=int(g["sims"]), seed=int(g["seed"]))
    plain = rt.run_job(pts, region, spec, rt.DeviceExecutor(device=0, comm=False))
    ex = rt.DeviceExecutor(device=0, comm=True)
    assert ex.comm and api["dev"].comm_rank() == (0, 1)
    try:
        coll = rt.run_job(pts, region, spec, ex)
    finally:
        api["dev"].comm_destroy()
    for a, b in ((plain.k_hat, coll.k_hat), (plain.l_hat, coll.l_hat),
                 (plain.upper_l, coll.upper_l), (plain.lower_l, coll.lower_l),
                 (plain.diff_upper, coll.diff_upper)):
        assert np.array_equal(a.values, b.values)
    assert coll.telemetry.in_threshold_pairs == plain.telemetry.in_threshold_pairs
    assert surfaces_close(coll.k_hat.values, g["k"], TOL)
    assert surfaces_close(coll.upper_l.values, g["upper"], TOL)


def test_invalid_point_raises_without_writing_outputs(api):
    """Validation runs on the device without a mid-call round trip; a point
    outside the region still raises the reference's invalid_argument
    (estimator.cpp:123-127) and leaves the caller's buffers untouched."""
    import ctypes as C

    from paper_1912_04753_b200 import _lib

    dev, est, geom = api["dev"], api["est"], api["geom"]
    ring, p0, p1 = square(1000.0, 0, 100)
    region = geom.StudyRegion(ring, p0, p1)
    grid = est.DistanceGrid([50.0, 100.0], [5, 10])
    dev.configure(region, grid)
    rng = np.random.default_rng(4)
    x = rng.uniform(0, 1000, 500); y = rng.uniform(0, 1000, 500); t = rng.integers(0, 101, 500)
    x[123] = 1500.0
    k = np.full((2, 2), 7.0)
    rc = dev.lib.stk_run_job(dev.h, _lib.ptr(x), _lib.ptr(y), _lib.ptr(t, C.c_int64), 500, 3, 1,
                             0, _lib.ptr(k), None, None, None, None, None)
    assert rc == _lib.STK_EINVAL
    assert dev.lib.stk_last_error(dev.h).decode() == "point outside study region or period"
    assert np.all(k == 7.0)
    t[5] = 101
    x[123] = 500.0
    with pytest.raises(ValueError, match="point outside study region or period"):
        est.estimate_surface((x, y, t), region, grid)
    t[5] = 100  # the context recovers: the next call is valid
    est.estimate_surface((x, y, t), region, grid)


def test_repeated_job_graph_replay_bit_identical(api):
    """The second identical call captures the pipeline as a CUDA graph and
    later calls replay it (one launch, one synchronisation): results stay bit
    for bit the same into fresh output buffers, the device timers keep
    working, and changing an argument (seed) runs the pipeline anew."""
    import ctypes as C

    from paper_1912_04753_b200 import _lib

    dev, est, geom, sim = api["dev"], api["est"], api["geom"], api["sim"]
    ring, p0, p1 = square(1000.0, 0, 365 * 86400)
    region = geom.StudyRegion(ring, p0, p1)
    grid = est.DistanceGrid.regular(10.0, 100.0, 3 * 86400, 30 * 86400)
    pts = sim.generate_cstr(10000, region, 1, device=0)
    dev.configure(region, grid)
    shape = (grid.cells_s(), grid.cells_t())

    def call(seed):
        outs = [np.full(shape, -1.0) for _ in range(5)]
        tel = _lib.StkTelemetry()
        dev.check(dev.lib.stk_run_job(dev.h, _lib.ptr(pts.x), _lib.ptr(pts.y),
                                      _lib.ptr(pts.t, C.c_int64), len(pts), 3, seed, 0,
                                      *[_lib.ptr(o) for o in outs], C.byref(tel)))
        return outs, tel

    first, t1 = call(5)
    for _ in range(4):  # plain, capture, replay, replay
        again, tn = call(5)
        for a, b in zip(first, again):
            assert np.array_equal(a, b)
        assert tn.in_threshold_pairs == t1.in_threshold_pairs
        assert tn.pair_ms > 0.0 and tn.total_ms > 0.0 and tn.kernel_launches == t1.kernel_launches
    other, to = call(6)
    assert not np.array_equal(other[2], first[2])  # different realisations: other envelopes
    assert to.in_threshold_pairs != t1.in_threshold_pairs


def test_parallel_permutation_bit_exact_large(api, port):
    """The parallel Fisher-Yates (perm_* kernels: swap targets from the MT
    stream in parallel, counting sort of the targets, short increasing
    chains) reproduces generate_permutation's sequential swaps
    (simulation.cpp:37-53) bit for bit at n = 200,000, and equals the
    sequential device kernel (STK_SEQ_PERMUTATION) run in a fresh process."""
    import ctypes as C

    from paper_1912_04753_b200 import _lib

    dev, geom = api["dev"], api["geom"]
    dev.configure(geom.StudyRegion([[0, 0], [1000, 0], [1000, 1000], [0, 1000]], 0, 10**9))
    rng = np.random.default_rng(12)
    n = 200_000
    x = rng.uniform(0, 1000, n); y = rng.uniform(0, 1000, n); t = rng.integers(0, 10**9, n)
    for seed in (3, 2**63 + 5):
        ox, oy, ot = np.zeros(n), np.zeros(n), np.zeros(n, np.int64)
        dev.check(dev.lib.stk_generate(dev.h, 2, n, _lib.ptr(x), _lib.ptr(y),
                                       _lib.ptr(t, C.c_int64), seed, _lib.ptr(ox), _lib.ptr(oy),
                                       _lib.ptr(ot, C.c_int64)))
        rx, ry, rt_ = port.generate_permutation(x, y, t, seed)
        assert np.array_equal(ox, rx) and np.array_equal(oy, ry) and np.array_equal(ot, rt_)
    code = (
        "import sys, numpy as np, ctypes as C; sys.path.insert(0, %r)\n"
        "from paper_1912_04753_b200 import _lib\n"
        "from paper_1912_04753_b200.stripley import device, geom\n"
        "d = device.get(0)\n"
        "d.configure(geom.StudyRegion([[0, 0], [1000, 0], [1000, 1000], [0, 1000]], 0, 10**9))\n"
        "r = np.random.default_rng(12); n = 200000\n"
        "x = r.uniform(0, 1000, n); y = r.uniform(0, 1000, n); t = r.integers(0, 10**9, n)\n"
        "o = [np.zeros(n), np.zeros(n), np.zeros(n, np.int64)]\n"
        "d.check(d.lib.stk_generate(d.h, 2, n, _lib.ptr(x), _lib.ptr(y), _lib.ptr(t, C.c_int64),"
        " 3, _lib.ptr(o[0]), _lib.ptr(o[1]), _lib.ptr(o[2], C.c_int64)))\n"
        "np.save(sys.argv[1], o[2])\n" % ROOT)
    with tempfile.TemporaryDirectory() as dd:
        out = os.path.join(dd, "t.npy")
        env = dict(os.environ, STK_SEQ_PERMUTATION="1")
        r = subprocess.run(["python", "-c", code, out], env=env, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr
        seq = np.load(out)
    rx, ry, rt_ = port.generate_permutation(x, y, t, 3)
    assert np.array_equal(seq, rt_)
