"""The reference's statistical acceptance criteria through the device path
(proj/tests/acceptance/acceptance_main.cpp).

* criterion 3 (:160-210): calibration on CSR — mean L over 100 realisations
  (seeds 3000 + r, the same draws as the reference's generate_cstr) within 3
  standard errors of 0 in every cell, and the reference plane 2 pi s^2 t;
* criterion 4 (:212-247): significance — the reference's clustered test pattern
  exceeds the upper envelope of 39 CSR simulations at cluster scale in at
  least 19 of 20 repetitions (rt::run_job with the reference's seeds).

Because the device CSR generator is bit-exact and K agrees with the reference
to ~1e-15, these statistics are the reference's own; the tests check that the
device pipeline (generation, pairs, finalize, L, envelope, diff) delivers them.
"""
import numpy as np
import pytest

from conftest import surfaces_close

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_1912_04753_b200.stripley import device, est, geom, rt, sim

    device.get(0)
    return dict(est=est, geom=geom, rt=rt, sim=sim)


def test_criterion3_csr_calibration(api):
    est, geom, sim = api["est"], api["geom"], api["sim"]
    ring = np.array([[0, 0], [2000, 0], [2000, 1000], [0, 1000]], float)
    region = geom.StudyRegion(ring, 0, 1_000_000)
    grid = est.DistanceGrid.regular(100.0, 400.0, 100_000, 400_000)
    pts = sim.generate_cstr(500, region, 1)  # unused by CSR realisations (shape only)
    runs = 100
    ls = sim.run_simulations(pts, region, grid, sim.Method.Cstr, runs, 3000)
    vals = np.stack([l.values for l in ls])
    mean = vals.mean(axis=0)
    se = np.sqrt(vals.var(axis=0, ddof=1) / runs)
    z = np.abs(mean) / se
    assert z.max() <= 3.0, f"worst |mean L| is {z.max():.2f} standard errors from 0"
    theo = est.theoretical_surface(grid)
    s = np.array(grid.s_values)[:, None]
    t = np.array(grid.t_values, dtype=float)[None, :]
    assert np.array_equal(theo.values, 2.0 * np.pi * s * s * t)


def test_criterion4_significance(api):
    from oracle import ref

    if not __import__("oracle").ref_available():
        pytest.skip("reference test helpers (oracle/_ref) not built")
    est, geom, rt = api["est"], api["geom"], api["rt"]
    side = 20000.0
    ring = np.array([[0, 0], [side, 0], [side, side], [0, side]], float)
    region = geom.StudyRegion(ring, 0, 50)
    grid = est.DistanceGrid.regular(250.0, 1000.0, 2, 6)
    detected = 0
    for rep in range(20):
        x, y, t = ref.clustered_points(400 + rep, ring, 0, 50, 2000, 5, 500.0, 2.0)
        spec = rt.JobSpec(grid=grid, sims=39, seed=4000 + 100 * rep)
        res = rt.run_job((x, y, t), region, spec, rt.DeviceExecutor(device=0))
        # cluster scale: spatial cells 1.. (sigma_s..2 sigma_s), every temporal cell
        if np.any(res.diff_upper.values[1:, :] > 0.0):
            detected += 1
    assert detected >= 19, f"clustering detected in only {detected}/20 repetitions"


def test_criterion9_smoke_benchmark_matches_reference(api):
    """Criterion 9 (:478-506): n = 10,000 uniform points (the reference's own
    generator, seed 909), 20 x 20 grid, 19 CSR simulations, seed 77 — well
    under the 5-minute bar, and equal to the reference's rt::run_job (K, L,
    envelopes, diff within 1e-9; in-threshold pairs of the observed pattern
    exact)."""
    import time

    from oracle import ref

    if not __import__("oracle").ref_available():
        pytest.skip("reference (oracle/_ref) not built")
    est, geom, rt = api["est"], api["geom"], api["rt"]
    side = 10000.0
    ring = np.array([[0, 0], [side, 0], [side, side], [0, side]], float)
    region = geom.StudyRegion(ring, 0, 100)
    grid = est.DistanceGrid.regular(25.0, 500.0, 2, 40)
    x, y, t = ref.uniform_points(909, ring, 0, 100, 10000)
    spec = rt.JobSpec(grid=grid, sims=19, seed=77)
    t0 = time.perf_counter()
    res = rt.run_job((x, y, t), region, spec, rt.DeviceExecutor(device=0))
    elapsed = time.perf_counter() - t0
    assert elapsed < 300.0
    assert res.k_hat.values.shape == (20, 20) and res.upper_l is not None
    r = ref.run_job(x, y, t, ring, 0, 100, grid.s_values, grid.t_values, 19, 77,
                    partitions=8, workers=4, use_index=True, use_cache=True)
    # observed + 19 realisations, the same total as the reference's (index-invariant)
    assert res.telemetry.in_threshold_pairs == r["in_threshold"]

    assert surfaces_close(res.k_hat.values, r["k"]) and surfaces_close(res.l_hat.values, r["l"])
    assert surfaces_close(res.upper_l.values, r["upper"])
    assert surfaces_close(res.lower_l.values, r["lower"])
    assert surfaces_close(res.diff_upper.values, r["diff"])
