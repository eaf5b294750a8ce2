"""CPU: pin the oracle before trusting it.

The C restatement (oracle/oracle.c, the "port") is checked against
* the reference's bundled golden output proj/data/sample_result.json
  (committed as tests/golden/sample_result.npz by tests/golden/make_golden.py),
* the reference's known-answer tests (test_edge_correction.cpp,
  test_estimator.cpp, test_simulation.cpp),
* the C++ standard's known answer for std::mt19937_64,
* fixtures produced by the reference compiled from its own sources, and —
  when oracle/_ref is built in this container — the reference live.
"""
import numpy as np
import pytest

import oracle
from conftest import golden, rel_err, surfaces_close
from oracle import port

SQUARE_10K = np.array([[0, 0], [10000, 0], [10000, 10000], [0, 10000]], float)


def test_mt19937_64_standard_known_answer():
    # C++ [rand.predef]: the 10000th invocation of a default-constructed
    # mt19937_64 (seed 5489) produces 9981545732273789042.
    out = port.mt_outputs(5489, 10000)
    assert int(out[-1]) == 9981545732273789042


def test_mt_stream_matches_reference_fixture():
    g = golden("mt19937_64.npz")
    for i, seed in enumerate(g["seeds"]):
        assert np.array_equal(port.mt_outputs(int(seed), 1000), g[f"s{i}"])


def test_golden_sample_result_through_port():
    """proj/data/sample_result.json: 1,000 points, 20x20 grid, 19 CSR sims, seed 42."""
    g = golden("sample_result.npz")
    x, y, t, ring = g["x"], g["y"], g["t"], g["ring"]
    s, tv = g["s"], g["tv"]
    obs = port.estimate(x, y, t, ring, 0, 365, s, tv)
    assert surfaces_close(obs["k"], g["k"], 1e-12)
    assert surfaces_close(obs["l"], g["l"], 1e-12)
    assert np.array_equal(obs["counts"], g["counts_observed"])
    ls = []
    total = obs["in_threshold"]
    for r in range(int(g["sims"])):
        sx, sy, st = port.generate_cstr(len(x), ring, 0, 365, int(g["seed"]) + r)
        e = port.estimate(sx, sy, st, ring, 0, 365, s, tv)
        ls.append(e["l"])
        total += e["in_threshold"]
    up, lo = port.envelopes(np.stack(ls))
    assert surfaces_close(up, g["upper"], 1e-12)
    assert surfaces_close(lo, g["lower"], 1e-12)
    assert surfaces_close(port.diff(obs["l"], up), g["diff"], 1e-12)
    assert total == int(g["in_threshold_total"])  # 1,048,148


def test_edge_correction_known_answers():
    """proj/tests/test_edge_correction.cpp:10-29 and :64-72."""
    w = port.spatial_weight
    assert w(5000, 5000, 1000, SQUARE_10K) == 1.0
    assert w(5000, 5000, 0.0, SQUARE_10K) == 1.0
    assert w(1500, 1500, 1499, SQUARE_10K) == pytest.approx(1.0)
    assert w(5000, 0, 100, SQUARE_10K) == pytest.approx(0.5)
    assert w(0, 5000, 250, SQUARE_10K) == pytest.approx(0.5)
    assert w(0, 0, 100, SQUARE_10K) == pytest.approx(0.25)
    assert w(10000, 10000, 400, SQUARE_10K) == pytest.approx(0.25)
    assert np.isnan(w(200, 50, 10, np.array([[0, 0], [100, 0], [100, 100], [0, 100]], float)))
    tw = port.temporal_weight
    assert tw(50, 10, 0, 100) == 1.0
    assert tw(5, 10, 0, 100) == 0.5
    assert tw(95, 10, 0, 100) == 0.5
    assert tw(10, 10, 0, 100) == 1.0
    assert tw(90, 10, 0, 100) == 1.0
    assert tw(50, 0, 0, 100) == 1.0


def test_spatial_weight_fixture_bitwise():
    """Port == reference bit for bit (same libm, same operation order)."""
    g = golden("weights.npz")
    for k in range(int(g["count"])):
        ring = g[f"{k}_ring"]
        for cx, cy, d, w in zip(g[f"{k}_cx"], g[f"{k}_cy"], g[f"{k}_d"], g[f"{k}_w"]):
            assert port.spatial_weight(cx, cy, d, ring) == w


def test_two_point_hand_value():
    """proj/tests/test_estimator.cpp:62-76: K = 5e9."""
    h = port.estimate(np.array([4000.0, 5000.0]), np.array([5000.0, 5000.0]),
                      np.array([50, 55]), SQUARE_10K, 0, 100, np.array([2000.0]), np.array([10]))
    assert h["k"][0, 0] == pytest.approx(5.0e9, rel=1e-15)


def test_polygon_fixtures_through_port():
    """Criterion-1 datasets: port counts == reference counts; K within 1e-9 of
    estimate_surface and brute_force_k (helpers.hpp:95-139)."""
    g = golden("polygons.npz")
    s, tv = g["s"], g["tv"]
    for rep in range(int(g["count"])):
        ring = g[f"{rep}_ring"]
        x, y, t = g[f"{rep}_x"], g[f"{rep}_y"], g[f"{rep}_t"]
        h = port.estimate(x, y, t, ring, 0, 60, s, tv)
        assert np.array_equal(h["counts"], g[f"{rep}_counts"]), rep
        assert h["in_threshold"] == int(g[f"{rep}_pairs"])
        assert surfaces_close(h["k"], g[f"{rep}_k"], 1e-9), rep
        assert surfaces_close(h["k"], g[f"{rep}_k_bf"], 1e-9), rep


def test_c1_fixture_through_port():
    from paper_1912_04753_b200 import configs

    cfg = configs.CONFIGS["C1"]
    s, tv = configs.grid_values(cfg)
    g = golden("c1.npz")
    x, y, t = port.generate_cstr(cfg.n, cfg.ring(), 0, cfg.period_s, cfg.seed)
    assert np.array_equal(x[:16], g["x_head"]) and np.array_equal(t[:16], g["t_head"])
    h = port.estimate(x, y, t, cfg.ring(), 0, cfg.period_s, s, tv)
    assert np.array_equal(h["counts"], g["counts"])
    assert h["in_threshold"] == int(g["pairs"])
    assert surfaces_close(h["k"], g["k"], 1e-9)


def test_bootstrap_permutation_generators_vs_reference():
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built here")
    from oracle import ref

    g = golden("sample_result.npz")
    x, y, t = g["x"], g["y"], g["t"]
    for seed in (1, 42):
        a = port.generate_bootstrap(x, y, t, seed)
        b = ref.generate_bootstrap(x, y, t, seed)
        assert all(np.array_equal(u, v) for u, v in zip(a, b))
        a = port.generate_permutation(x, y, t, seed)
        b = ref.generate_permutation(x, y, t, seed)
        assert all(np.array_equal(u, v) for u, v in zip(a, b))


def test_port_vs_live_reference_random_polygons():
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built here")
    from oracle import ref

    s, tv = ref.regular_grid(150.0, 600.0, 10, 40)
    for rep in range(6):
        ring = (ref.random_convex_ring(17 + rep, 800.0, 600.0, 9) if rep % 2 == 0
                else ref.random_star_ring(17 + rep, 700.0, 11))
        x, y, t = ref.uniform_points(90 + rep, ring, 0, 60, 60 + 20 * rep)
        k_ref, pairs, _ = ref.estimate_surface(x, y, t, ring, 0, 60, s, tv, use_index=True)
        h = port.estimate(x, y, t, ring, 0, 60, s, tv)
        assert h["in_threshold"] == pairs
        assert rel_err(h["k"], k_ref) <= 1e-12
        assert np.array_equal(h["counts"], ref.pair_counts(x, y, t, s, tv))


def test_fixed_point_rounding():
    # 53 fractional bits: 2^53 is 1.0; 2 + 2^-53 rounds to 2; hi words round once.
    assert port.__name__  # noqa
    lib = oracle._load_port()
    assert lib.orc_fixed_to_double(0, 1 << 53) == 1.0
    assert lib.orc_fixed_to_double(1, 0) == 2.0 ** 11
    assert lib.orc_fixed_to_double(0, (1 << 54) + 1) == 2.0
    assert lib.orc_fixed_to_double(0, (1 << 53) - 1) == 1.0 - 2.0 ** -53  # a term below 1


def test_port_vs_live_reference_degenerate_weights():
    """Reference rounding corners the port must reproduce: omega == 0 (the
    circle through all four corners of a square: 1/0 enters the bin, whose K
    is NaN in the reference) and omega slightly above 1 (an arc sum one ulp
    over 2*pi at UTM-like coordinates: a term just below 1)."""
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built here")
    from oracle import ref

    ring = np.array([[0, 0], [100.0, 0], [100.0, 100.0], [0, 100.0]])
    x = np.array([0.0, 0.0, 50.0, 50.0, 50.0, 100.0])
    t = np.array([0, 0, 10, 10, 12, 100])
    s, tv = np.array([1.0, 10.0, 200.0]), np.array([1, 5, 100], np.int64)
    k_ref, _, _ = ref.estimate_surface(x, x.copy(), t, ring, 0, 100, s, tv, use_index=True)
    h = port.estimate(x, x.copy(), t, ring, 0, 100, s, tv)
    assert np.isnan(k_ref[2, 2]) and surfaces_close(h["k"], k_ref, 1e-12)
    # omega = 1 + 2^-52 from the reference (found by tests/test_gpu_polygons.py)
    a = 2.0 * np.pi * np.arange(200) / 200
    r = 1000.0 * np.random.default_rng(4).uniform(0.4, 1.0, 200)
    star = np.stack([1100.0 + r * np.cos(a), 1100.0 + r * np.sin(a)], axis=1) + [4.5e5, 4.2e6]
    w = ref.spatial_weight(451257.7456706156, 4200906.479450759, 173.86844087028163, star)
    assert w == port.spatial_weight(451257.7456706156, 4200906.479450759, 173.86844087028163,
                                    star)
    cx, cy = 451103.41905628354, 4200826.394927663
    assert ref.spatial_weight(cx, cy, 173.86844087028163, star) > 1.0  # 1 + 2^-52
    xs = np.array([cx, 451257.7456706156])
    ys = np.array([cy, 4200906.479450759])
    ts = np.array([227, 251])
    s2, tv2 = np.array([150.0, 300.0]), np.array([50, 400], np.int64)
    k_ref, _, _ = ref.estimate_surface(xs, ys, ts, star, 0, 400, s2, tv2, use_index=True)
    h = port.estimate(xs, ys, ts, star, 0, 400, s2, tv2)
    assert rel_err(h["k"], k_ref) <= 1e-15


def test_reference_job_split_per_pattern_reproduces_run_job():
    """oracle.ref.Job (ref_job_open / ref_job_pattern: rt::run_job's loop body
    split per pattern, the path the large fixtures and the bench's reference
    arm use) reproduces the reference's own golden sample bit for bit, and the
    R-tree per-bin counts equal the O(n^2) ones."""
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built here")
    from oracle import ref

    g = golden("sample_result.npz")
    x, y, t, ring = g["x"], g["y"], g["t"], g["ring"]
    job = ref.Job(x, y, t, ring, 0, 365, g["s"], g["tv"], seed=int(g["seed"]), partitions=1,
                  workers=1, use_cache=True)
    obs = job.pattern(-1)
    assert np.array_equal(obs["k"], g["k"]) and np.array_equal(obs["l"], g["l"])
    ls, total = [], obs["in_threshold"]
    for r in range(int(g["sims"])):
        p = job.pattern(r)
        ls.append(p["l"])
        total += p["in_threshold"]
    job.close()
    assert np.array_equal(np.max(ls, 0), g["upper"]) and np.array_equal(np.min(ls, 0), g["lower"])
    assert total == int(g["in_threshold_total"])
    c_idx = ref.pair_counts_indexed(x, y, t, g["s"], g["tv"], threads=4)
    assert np.array_equal(c_idx, ref.pair_counts(x, y, t, g["s"], g["tv"]))
    assert np.array_equal(c_idx, g["counts_observed"])


def test_large_fixtures_consistent():
    """The committed full-size fixtures agree with themselves: per-bin counts
    sum to the reference's in-threshold totals; C3 has every ordered pair in
    threshold; subset envelopes are the max / min of their realisations."""
    import os

    from conftest import GOLDEN

    if os.path.exists(os.path.join(GOLDEN, "c2_job.npz")):
        g = golden("c2_job.npz")
        assert int(g["counts_observed"].sum()) == int(g["in_threshold_observed"])
        assert int(g["in_threshold_total"]) > int(g["in_threshold_observed"])
    if os.path.exists(os.path.join(GOLDEN, "c3_full.npz")):
        g = golden("c3_full.npz")
        n = int(g["n"])
        assert int(g["counts"].sum()) == int(g["in_threshold"]) == n * (n - 1)
    for name in ("c4_parity.npz", "c5_parity.npz"):
        if not os.path.exists(os.path.join(GOLDEN, name)):
            continue
        g = golden(name)
        rs = [int(r) for r in g["realisations"]]
        for key in ["obs"] + [f"r{r}" for r in rs]:
            if f"{key}_counts" in g.files:
                assert int(g[f"{key}_counts"].sum()) == int(g[f"{key}_in_threshold"])
        if "upper_subset" in g.files:
            ls = np.stack([g[f"r{r}_l"] for r in rs])
            assert np.array_equal(ls.max(0), g["upper_subset"])
            assert np.array_equal(ls.min(0), g["lower_subset"])
