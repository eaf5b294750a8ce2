"""GPU parity for general polygons at scale: the slab
point-in-polygon, the edge-cell lists of the arc weight and safe radius, and
the parallel rejection-sampling CSR generator, against the oracle port (the C
restatement pinned to the reference in tests/test_oracle_cpu.py).

Rings follow the reference's acceptance criterion 6 (a circle of 128..2,048
vertices, proj/tests/acceptance/acceptance_main.cpp:295-303) plus random star
polygons (proj/tests/helpers.hpp:40-50).  Bars as everywhere: generated points
and counts bit-exact, weights <= 1e-12, K <= 1e-9 relative.
"""
import numpy as np
import pytest

from conftest import golden, rel_err, surfaces_close

pytestmark = pytest.mark.gpu

TOL = 1e-9


@pytest.fixture(scope="module")
def api():
    from paper_1912_04753_b200.stripley import device, est, geom, sim

    device.get(0)
    return dict(est=est, geom=geom, sim=sim, dev=device.get(0))


@pytest.fixture(scope="module")
def port():
    from oracle import port

    return port


def circle_ring(v, r=5000.0, cx=5000.0, cy=5000.0):
    a = 2.0 * np.pi * np.arange(v) / v
    return np.stack([cx + r * np.cos(a), cy + r * np.sin(a)], axis=1)


def star_ring(v, seed, radius=1000.0):
    rng = np.random.default_rng(seed)
    a = 2.0 * np.pi * np.arange(v) / v
    r = radius * rng.uniform(0.4, 1.0, v)
    return np.stack([radius * 1.1 + r * np.cos(a), radius * 1.1 + r * np.sin(a)], axis=1)


RINGS = {
    "circle2048": circle_ring(2048),
    "circle128": circle_ring(128),
    "star300": star_ring(300, 3),
    "offset_star": star_ring(200, 4) + np.array([4.5e5, 4.2e6]),  # UTM-like coordinates
}


@pytest.mark.parametrize("name", sorted(RINGS))
def test_parallel_polygon_csr_bit_exact(api, port, name):
    """csr_poly_kernel (parallel starts + chain walk) == generate_cstr's stream."""
    sim, geom = api["sim"], api["geom"]
    ring = RINGS[name]
    for (p0, p1), seed, n in [((0, 365 * 86400), 1, 20_000), ((0, 60), 7, 1),
                              ((-5, 5), 2**63 + 11, 4_097), ((0, 2**62 + 12_345), 3, 3_000)]:
        region = geom.StudyRegion(ring, p0, p1)
        pts = sim.generate_cstr(n, region, seed)
        x, y, t = port.generate_cstr(n, ring, p0, p1, seed)
        assert np.array_equal(pts.x, x) and np.array_equal(pts.y, y), (name, seed)
        assert np.array_equal(pts.t, t), (name, seed)


def test_many_realisations_polygon_csr(api, port):
    """A batch of realisations (one CTA each) through run_simulations' seed ladder."""
    sim, geom = api["sim"], api["geom"]
    ring = RINGS["circle128"]
    region = geom.StudyRegion(ring, 0, 1000)
    for r in (0, 5, 63):
        pts = sim.generate_cstr(2_000, region, 100 + r)
        x, y, t = port.generate_cstr(2_000, ring, 0, 1000, 100 + r)
        assert np.array_equal(pts.x, x) and np.array_equal(pts.t, t)


@pytest.mark.parametrize("name", ["circle2048", "star300", "offset_star"])
def test_polygon_weights_through_edge_cells(api, port, name):
    """stk_spatial_weights with a grid set (edge cells active for d <= s_max)
    and beyond s_max (full ring), against the port."""
    est, geom, dev = api["est"], api["geom"], api["dev"]
    from paper_1912_04753_b200 import _lib

    ring = RINGS[name]
    region = geom.StudyRegion(ring, 0, 100)
    span = float(np.ptp(ring[:, 0]))
    grid = est.DistanceGrid([0.05 * span, 0.1 * span, 0.2 * span], [10, 100])
    dev.configure(region, grid)
    rng = np.random.default_rng(5)
    xmin, ymin = ring.min(0)
    xmax, ymax = ring.max(0)
    cx, cy = [], []
    while len(cx) < 600:
        px, py = rng.uniform(xmin, xmax), rng.uniform(ymin, ymax)
        if port.point_in_polygon(px, py, ring):
            cx.append(px)
            cy.append(py)
    cx, cy = np.array(cx), np.array(cy)
    d = np.concatenate([rng.uniform(0.0, 0.2 * span, 400), rng.uniform(0.2 * span, span, 200)])
    want = np.array([port.spatial_weight(a, b, c, ring) for a, b, c in zip(cx, cy, d)])
    w = np.zeros_like(want)
    dev.check(dev.lib.stk_spatial_weights(dev.h, _lib.ptr(cx), _lib.ptr(cy), _lib.ptr(d), len(cx),
                                          _lib.ptr(w)))
    assert np.array_equal(w == 1.0, want == 1.0), name
    assert rel_err(w, want) <= 1e-12, name


@pytest.mark.parametrize("name,n,frac", [("circle2048", 1200, 0.15), ("circle128", 3000, 0.1),
                                         ("star300", 1000, 0.3), ("offset_star", 1000, 0.3)])
def test_polygon_pair_histogram_and_k(api, port, name, n, frac):
    """Counts bit-exact, weighted sums ~1e-13, K <= 1e-9: pair kernel with the
    edge-cell arc weight, slab PIP probes and list-bounded safe radii."""
    est, geom, sim = api["est"], api["geom"], api["sim"]
    ring = RINGS[name]
    p0, p1 = 0, 400
    region = geom.StudyRegion(ring, p0, p1)
    pts = sim.generate_cstr(n, region, 17)
    span = float(np.ptp(ring[:, 0]))
    s = np.array([frac * span * f for f in (0.25, 0.5, 0.75, 1.0)])
    tv = np.array([50, 150, 400], np.int64)
    grid = est.DistanceGrid(s, tv)
    h = est.pair_histogram(pts, region, grid)
    o = port.pair_histogram(pts.x, pts.y, pts.t, ring, p0, p1, s, tv)
    assert np.array_equal(h["counts"], o["counts"]), name
    assert rel_err(h["hist"], o["hist"]) <= 1e-13, name
    k = est.estimate_surface(pts, region, grid)
    ko = port.finalize(o["hist"], n, port.area(ring), p1 - p0)
    assert surfaces_close(k.values, ko, TOL), name


def test_polygon_boundary_centers_and_validation(api, port):
    """Centers on vertices and edges of a 2,048-gon (on_segment through the
    slab PIP), and the reference's error for a point just outside."""
    est, geom = api["est"], api["geom"]
    ring = RINGS["circle2048"]
    region = geom.StudyRegion(ring, 0, 100)
    k = np.arange(0, 2048, 97)
    mid = 0.5 * (ring[k] + ring[(k + 1) % 2048])
    rng = np.random.default_rng(9)
    inner = 5000.0 + (rng.uniform(0, 4000, (60, 2)) - 2000.0)
    xy = np.concatenate([ring[k], mid, inner])
    t = rng.integers(0, 101, len(xy))
    s = np.array([250.0, 500.0, 1000.0, 3000.0])
    tv = np.array([20, 100], np.int64)
    grid = est.DistanceGrid(s, tv)
    h = est.pair_histogram((xy[:, 0], xy[:, 1], t), region, grid)
    o = port.pair_histogram(xy[:, 0], xy[:, 1], t, ring, 0, 100, s, tv)
    assert np.array_equal(h["counts"], o["counts"])
    assert rel_err(h["hist"], o["hist"]) <= 1e-13
    # just outside an edge's midpoint (outward normal) -> the reference's message
    out = mid[3] * (1.0 + 1e-6) - 5000.0 * 1e-6
    with pytest.raises(ValueError, match="point outside study region"):
        est.estimate_surface((np.array([5000.0, out[0]]), np.array([5000.0, out[1]]),
                              np.array([0, 0])), region, grid)


def test_golden_polygons_still_exact(api, port):
    """The criterion-1 golden polygons (reference outputs) through the new path."""
    est, geom = api["est"], api["geom"]
    g = golden("polygons.npz")
    grid = est.DistanceGrid(g["s"], g["tv"])
    for rep in range(0, int(g["count"]), 3):
        ring = g[f"{rep}_ring"]
        region = geom.StudyRegion(ring, 0, 60)
        pts = (g[f"{rep}_x"], g[f"{rep}_y"], g[f"{rep}_t"])
        k = est.estimate_surface(pts, region, grid)
        assert surfaces_close(k.values, g[f"{rep}_k"], TOL), rep
