"""Regenerate the golden fixtures in tests/golden/ from the reference itself.

Run HERE (the container that has /root/reference):  python tests/golden/make_golden.py
The fixtures are what the GPU-box tests compare against (the reference tree
does not exist there).  Every array is produced by the reference compiled from
its own sources (oracle/_ref) or read from its bundled golden output
(proj/data/sample_result.json); nothing is hand-written.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from oracle import ref  # noqa: E402
from paper_1912_04753_b200 import configs  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
DATA = "/root/reference/proj/data"


def sample():
    d = json.load(open(os.path.join(DATA, "sample_result.json")))
    rows = [l.strip().split(",") for l in open(os.path.join(DATA, "sample_points.csv")).read().strip().split("\n")[1:]]
    x = np.array([float(r[1]) for r in rows])
    y = np.array([float(r[2]) for r in rows])
    t = np.array([int(r[3]) for r in rows], dtype=np.int64)
    ring = np.array([[0, 0], [10000, 0], [10000, 10000], [0, 10000]], float)  # sample_boundary.wkt
    s, tv = ref.regular_grid(100, 2000, 5, 100)
    r = ref.run_job(x, y, t, ring, 0, 365, s, tv, sims=19, seed=42, partitions=1, workers=1,
                    use_index=True, use_cache=True)
    golden = dict(k=np.array(d["k_hat"]), l=np.array(d["l_hat"]),
                  upper=np.array(d["envelope"]["upper_l"]), lower=np.array(d["envelope"]["lower_l"]),
                  diff=np.array(d["diff_upper"]))
    for k, v in golden.items():  # the reference reproduces its own golden file bit-exactly
        assert np.array_equal(r[k], v), k
    assert r["in_threshold"] == d["telemetry"]["comparisons"]["in_threshold_pairs"]
    counts = ref.pair_counts(x, y, t, s, tv)
    np.savez_compressed(os.path.join(OUT, "sample_result.npz"), x=x, y=y, t=t, ring=ring,
                        p0=0, p1=365, s=s, tv=tv, sims=19, seed=42,
                        in_threshold_total=r["in_threshold"], counts_observed=counts, **golden)


def polygons(count=24):
    """Criterion-1 style datasets (tests/acceptance/acceptance_main.cpp:45-78)."""
    sets = {}
    s, tv = ref.regular_grid(120.0, 360.0, 12, 36)
    for rep in range(count):
        if rep % 2 == 0:
            ring = ref.random_convex_ring(1000 + rep, 900.0, 700.0, 10)
        else:
            ring = ref.random_star_ring(1000 + rep, 800.0, 14)
        n = int(10 + (rep * 37) % 290)
        if rep % 3 == 0:
            x, y, t = ref.clustered_points(2000 + rep, ring, 0, 60, n, 4, 90.0, 5.0)
        else:
            x, y, t = ref.uniform_points(2000 + rep, ring, 0, 60, n)
        k_idx, pairs, _ = ref.estimate_surface(x, y, t, ring, 0, 60, s, tv, use_index=True)
        k_bf = ref.brute_force_k(x, y, t, ring, 0, 60, s, tv)
        counts = ref.pair_counts(x, y, t, s, tv)
        for key, v in dict(ring=ring, x=x, y=y, t=t, k=k_idx, k_bf=k_bf, counts=counts,
                           pairs=pairs).items():
            sets[f"{rep}_{key}"] = v
    np.savez_compressed(os.path.join(OUT, "polygons.npz"), s=s, tv=tv, count=count, **sets)


def weights():
    """(center, d) -> omega from edge::spatial_isotropic_weight on squares and stars."""
    rng = np.random.default_rng(5)
    out = {}
    rings = [np.array([[0, 0], [10000, 0], [10000, 10000], [0, 10000]], float),
             ref.random_star_ring(77, 1000.0, 12), ref.random_convex_ring(78, 900, 700, 10),
             ref.random_star_ring(79, 800.0, 64)]
    for k, ring in enumerate(rings):
        xmin, ymin = ring.min(0)
        xmax, ymax = ring.max(0)
        cx, cy, dd, ww = [], [], [], []
        while len(cx) < 400:
            px, py = rng.uniform(xmin, xmax), rng.uniform(ymin, ymax)
            if not ref.point_in_polygon(px, py, ring):
                continue
            d = rng.uniform(0.0, 0.9 * max(xmax - xmin, ymax - ymin))
            cx.append(px); cy.append(py); dd.append(d)
            ww.append(ref.spatial_weight(px, py, d, ring))
        out[f"{k}_ring"] = ring
        out[f"{k}_cx"] = np.array(cx); out[f"{k}_cy"] = np.array(cy)
        out[f"{k}_d"] = np.array(dd); out[f"{k}_w"] = np.array(ww)
    np.savez_compressed(os.path.join(OUT, "weights.npz"), count=len(rings), **out)


def rect_stress():
    """Rectangle (center, d) cases around the single-edge closed form's gates:
    circles just reaching one edge (d/h - 1 from 1e-15 to 1), just missing it,
    near corners, tiny radii, and regions at large coordinate offsets."""
    rng = np.random.default_rng(11)
    out = {}
    rects = [(0.0, 0.0, 10000.0, 10000.0), (500000.0, 4000000.0, 550000.0, 4030000.0),
             (-3.5, 2.25, 1.5, 9.0), (0.0, 0.0, 100000.0, 100000.0)]
    for k, (x0, y0, x1, y1) in enumerate(rects):
        ring = np.array([[x0, y0], [x1, y0], [x1, y1], [x0, y1]], float)
        W, H = x1 - x0, y1 - y0
        cx, cy, dd, ww = [], [], [], []
        while len(cx) < 1500:
            edge = rng.integers(4)
            h = W * 10.0 ** rng.uniform(-7, -0.4)
            along = rng.uniform(0.0, 1.0)
            if edge == 0:
                px, py = x0 + h, y0 + along * H
            elif edge == 1:
                px, py = x1 - h, y0 + along * H
            elif edge == 2:
                px, py = x0 + along * W, y0 + h
            else:
                px, py = x0 + along * W, y1 - h
            if not (x0 < px < x1 and y0 < py < y1):
                continue
            h_true = min(px - x0, x1 - px, py - y0, y1 - py)
            mode = rng.integers(4)
            if mode == 0:
                d = h_true * (1.0 + 10.0 ** rng.uniform(-15, 0))
            elif mode == 1:
                d = h_true * (1.0 - 10.0 ** rng.uniform(-15, -1))
            elif mode == 2:
                d = h_true * rng.uniform(1.0, 3.0)
            else:
                d = h_true + 10.0 ** rng.uniform(-12, 0) * max(abs(x0), abs(x1), 1.0) * 1e-3
            cx.append(px); cy.append(py); dd.append(d)
            ww.append(ref.spatial_weight(px, py, d, ring))
        out[f"{k}_ring"] = ring
        out[f"{k}_cx"] = np.array(cx); out[f"{k}_cy"] = np.array(cy)
        out[f"{k}_d"] = np.array(dd); out[f"{k}_w"] = np.array(ww)
    np.savez_compressed(os.path.join(OUT, "rect_stress.npz"), count=len(rects), **out)


def rect_corner_stress():
    """Rectangle (center, d) cases for the multi-side closed form: circles
    through or near corners (|K - c| -/+ tiny), containing 1..4 corners, and
    regions at large offsets."""
    rng = np.random.default_rng(12)
    out = {}
    rects = [(0.0, 0.0, 1000.0, 1000.0), (500000.0, 4000000.0, 503000.0, 4001000.0),
             (-2.0, -1.0, 2.0, 7.0)]
    for k, (x0, y0, x1, y1) in enumerate(rects):
        ring = np.array([[x0, y0], [x1, y0], [x1, y1], [x0, y1]], float)
        W, H = x1 - x0, y1 - y0
        corners = np.array([[x0, y0], [x1, y0], [x1, y1], [x0, y1]])
        cx, cy, dd, ww = [], [], [], []
        while len(cx) < 1500:
            px = x0 + W * rng.uniform(0.001, 0.999)
            py = y0 + H * rng.uniform(0.001, 0.999)
            mode = rng.integers(3)
            if mode == 0:    # near a corner distance
                kd = np.hypot(*(corners[rng.integers(4)] - [px, py]))
                d = kd * (1.0 + rng.choice([-1, 1]) * 10.0 ** rng.uniform(-14, -2))
            elif mode == 1:  # large circles: several sides, some corners inside
                d = rng.uniform(0.2, 1.5) * np.hypot(W, H)
            else:            # two nearby sides
                d = rng.uniform(0.5, 1.2) * (min(px - x0, x1 - px) + min(py - y0, y1 - py))
            cx.append(px); cy.append(py); dd.append(d)
            ww.append(ref.spatial_weight(px, py, d, ring))
        out[f"{k}_ring"] = ring
        out[f"{k}_cx"] = np.array(cx); out[f"{k}_cy"] = np.array(cy)
        out[f"{k}_d"] = np.array(dd); out[f"{k}_w"] = np.array(ww)
    np.savez_compressed(os.path.join(OUT, "rect_corner.npz"), count=len(rects), **out)


def rect_probe_free():
    """Rectangle (center, d) cases at the boundaries of the multi-side closed
    form's probe-free gates (stk_device.cuh rect_multi_edge_weight): corners at
    |g| / d^2 around 1e-4 on both sides, crossing sides with w / d around 1e-3,
    centers within 1e-9..1e-3 d of a side, thin rectangles, large offsets."""
    rng = np.random.default_rng(23)
    out = {}
    rects = [(0.0, 0.0, 1000.0, 1000.0), (0.0, 0.0, 1000.0, 3.0),
             (500000.0, 4000000.0, 501000.0, 4000700.0), (-50.0, -20.0, 50.0, 80.0)]
    for k, (x0, y0, x1, y1) in enumerate(rects):
        ring = np.array([[x0, y0], [x1, y0], [x1, y1], [x0, y1]], float)
        W, H = x1 - x0, y1 - y0
        corners = np.array([[x0, y0], [x1, y0], [x1, y1], [x0, y1]])
        cx, cy, dd, ww = [], [], [], []
        while len(cx) < 1200:
            px = x0 + W * rng.uniform(0.0005, 0.9995)
            py = y0 + H * rng.uniform(0.0005, 0.9995)
            mode = rng.integers(4)
            if mode == 0:    # |K - c|^2 - d^2 = +-eps d^2, eps around the 1e-4 gate
                kd2 = np.sum((corners[rng.integers(4)] - [px, py]) ** 2)
                eps = rng.choice([-1, 1]) * 10.0 ** rng.uniform(-5, -2)
                d = np.sqrt(kd2 / (1.0 + eps))
            elif mode == 1:  # a crossing side with w / d around 1e-3, plus larger circles
                h = [px - x0, x1 - px, py - y0, y1 - py][rng.integers(4)]
                wr = 10.0 ** rng.uniform(-4, -2)
                d = h / np.sqrt(1.0 - wr * wr) * (rng.uniform(1.0, 3.0) if rng.random() < 0.2 else 1.0)
            elif mode == 2:  # center within 1e-9..1e-3 d of a side, circle over corners
                d = rng.uniform(0.3, 1.5) * np.hypot(W, H)
                off = d * 10.0 ** rng.uniform(-9, -3)
                side = rng.integers(4)
                if side == 0: px = x0 + off
                elif side == 1: px = x1 - off
                elif side == 2: py = y0 + off
                else: py = y1 - off
            else:            # circles larger than the region
                d = rng.uniform(0.5, 2.0) * np.hypot(W, H)
            cx.append(px); cy.append(py); dd.append(d)
            ww.append(ref.spatial_weight(px, py, d, ring))
        out[f"{k}_ring"] = ring
        out[f"{k}_cx"] = np.array(cx); out[f"{k}_cy"] = np.array(cy)
        out[f"{k}_d"] = np.array(dd); out[f"{k}_w"] = np.array(ww)
    np.savez_compressed(os.path.join(OUT, "rect_probe_free.npz"), count=len(rects), **out)


def c1():
    """C1 (configs[0]) through the reference: K, per-bin counts, in_threshold."""
    cfg = configs.CONFIGS["C1"]
    s, tv = configs.grid_values(cfg)
    ring = cfg.ring()
    x, y, t = ref.generate_cstr(cfg.n, ring, 0, cfg.period_s, cfg.seed)
    k, pairs, _ = ref.estimate_surface(x, y, t, ring, 0, cfg.period_s, s, tv, use_index=True)
    counts = ref.pair_counts(x, y, t, s, tv)
    np.savez_compressed(os.path.join(OUT, "c1.npz"), k=k, counts=counts, pairs=pairs, s=s, tv=tv,
                        x_head=x[:16], t_head=t[:16])


def mt():
    seeds = [1, 42, 5489, 2**63 + 12345]
    np.savez_compressed(os.path.join(OUT, "mt19937_64.npz"), seeds=np.array(seeds, np.uint64),
                        **{f"s{i}": ref.mt_outputs(sd, 1000) for i, sd in enumerate(seeds)})


if __name__ == "__main__":
    oracle.build(with_ref=True)
    only = sys.argv[1:]
    jobs = dict(sample=sample, polygons=polygons, weights=weights, rect_stress=rect_stress,
                rect_corner=rect_corner_stress, rect_probe_free=rect_probe_free, c1=c1, mt=mt)
    for name, fn in jobs.items():
        if not only or name in only:
            fn()
    print("golden fixtures written to", OUT)
