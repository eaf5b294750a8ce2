"""The five BASELINE.json configurations as seeded synthetic inputs.

No public dataset is involved (the paper's Hubei data is unavailable).  Time
is integer seconds (the reference's ``STPoint::start_time`` is int64;
SURVEY §0.5): every config's temporal step is a whole number of seconds.
Regions are axis-aligned rectangles with period [0, extent].

* C1 uses the reference's own CSR generator (``generate_cstr(N, region, 1)``,
  MT19937-64) — on the device or, for checking, the oracle.
* C2 (Thomas) and C4/C5 (clusters + background) use numpy's PCG64 seeded with
  the config seed; points outside the window are redrawn so N is exact for
  C4/C5 and Poisson for C2, as the configs state.
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass

import numpy as np

DAY = 86400


@dataclass(frozen=True)
class Config:
    name: str
    n: int              # target N (C2: expected N of the Poisson process)
    extent_m: float     # square side
    period_s: int       # study period [0, period_s]
    s_step: float
    s_max: float
    t_step: int
    t_max: int
    sims: int
    seed: int
    kind: str           # csr | thomas | poi | uniform
    ring_vertices: int = 0  # > 0: a regular polygon inscribed in the square (acceptance c6 shape)

    def ring(self):
        e = self.extent_m
        if self.ring_vertices > 0:
            return circle_ring(self.ring_vertices, e)
        return np.array([[0.0, 0.0], [e, 0.0], [e, e], [0.0, e]])

    def with_ring(self, vertices: int) -> "Config":
        return dataclasses.replace(self, ring_vertices=int(vertices))


def circle_ring(vertices: int, extent: float):
    """Regular ``vertices``-gon inscribed in the circle of radius extent/2 around
    the square's center: the shape of the reference's acceptance criterion 6
    (proj/tests/acceptance/acceptance_main.cpp:295-303), scaled to the square."""
    a = 2.0 * np.pi * np.arange(vertices) / vertices
    h = 0.5 * extent
    return np.stack([h + h * np.cos(a), h + h * np.sin(a)], axis=1)


def inside_ring_strict(cfg: "Config", x, y):
    """Synthetic-data filter: points well inside the polygon (inside its
    inscribed circle, radius h*cos(pi/V), less a relative margin)."""
    if cfg.ring_vertices <= 0:
        return np.ones(len(x), bool)
    h = 0.5 * cfg.extent_m
    r_in = h * np.cos(np.pi / cfg.ring_vertices) * (1.0 - 1e-9)
    return (x - h) ** 2 + (y - h) ** 2 < r_in * r_in


CONFIGS = {
    "C1": Config("C1", 10_000, 1_000.0, 365 * DAY, 10.0, 100.0, 3 * DAY, 30 * DAY, 0, 1, "csr"),
    "C2": Config("C2", 100_000, 10_000.0, 365 * DAY, 50.0, 1_000.0, 129_600, 30 * DAY, 99, 2,
                 "thomas"),
    "C3": Config("C3", 200_000, 1_000.0, 100 * DAY, 93.75, 1_500.0, 540_000, 100 * DAY, 0, 3,
                 "csr"),
    "C4": Config("C4", 1_000_000, 50_000.0, 730 * DAY, 80.0, 2_000.0, 207_360, 60 * DAY, 99, 4,
                 "poi"),
    "C5": Config("C5", 10_000_000, 100_000.0, 1825 * DAY, 100.0, 5_000.0, 51_840, 30 * DAY, 199,
                 5, "poi"),
}


def grid_values(cfg: Config):
    """est::DistanceGrid::regular (estimator.cpp:24-32), accumulating s."""
    s_vals, s = [], cfg.s_step
    while s <= cfg.s_max * (1.0 + 1e-12):
        s_vals.append(s)
        s += cfg.s_step
    t_vals = list(range(cfg.t_step, cfg.t_max + 1, cfg.t_step))
    return np.array(s_vals), np.array(t_vals, dtype=np.int64)


def thomas(cfg: Config, parents=200, mean_offspring=500, sigma_s=50.0, sigma_t_days=5.0):
    """C2: space-time Thomas process; out-of-window offspring dropped."""
    rng = np.random.default_rng(cfg.seed)
    e, P = cfg.extent_m, cfg.period_s
    px = rng.uniform(0, e, parents)
    py = rng.uniform(0, e, parents)
    pt = rng.uniform(0, P, parents)
    k = rng.poisson(mean_offspring, parents)
    cx = np.repeat(px, k) + rng.normal(0, sigma_s, k.sum())
    cy = np.repeat(py, k) + rng.normal(0, sigma_s, k.sum())
    ct = np.floor(np.repeat(pt, k) + rng.normal(0, sigma_t_days * DAY, k.sum())).astype(np.int64)
    keep = (cx >= 0) & (cx <= e) & (cy >= 0) & (cy <= e) & (ct >= 0) & (ct <= P)
    return cx[keep], cy[keep], ct[keep]


def poi(cfg: Config, clusters=2000, frac_clustered=0.7):
    """C4/C5: 70% from log-normal(5,1)-sized Gaussian clusters (sigma_s ~ U(20,200) m,
    sigma_t ~ U(1,10) d) + 30% uniform background; exact N."""
    rng = np.random.default_rng(cfg.seed)
    e, P, n = cfg.extent_m, cfg.period_s, cfg.n
    n_cl = int(round(frac_clustered * n))
    sizes = rng.lognormal(5.0, 1.0, clusters)
    sizes = np.floor(sizes / sizes.sum() * n_cl).astype(np.int64)
    short = int(n_cl - sizes.sum())
    np.add.at(sizes, rng.choice(clusters, size=short, replace=True), 1)
    cxs = rng.uniform(0, e, clusters)
    cys = rng.uniform(0, e, clusters)
    cts = rng.uniform(0, P, clusters)
    ss = rng.uniform(20.0, 200.0, clusters)
    st = rng.uniform(1.0, 10.0, clusters) * DAY
    lab = np.repeat(np.arange(clusters), sizes)
    x = np.empty(n_cl)
    y = np.empty(n_cl)
    t = np.empty(n_cl, np.int64)
    todo = np.arange(n_cl)
    while len(todo):
        L = lab[todo]
        xx = cxs[L] + rng.normal(0, 1, len(todo)) * ss[L]
        yy = cys[L] + rng.normal(0, 1, len(todo)) * ss[L]
        tt = np.floor(cts[L] + rng.normal(0, 1, len(todo)) * st[L]).astype(np.int64)
        ok = (xx >= 0) & (xx <= e) & (yy >= 0) & (yy <= e) & (tt >= 0) & (tt <= P)
        x[todo[ok]] = xx[ok]
        y[todo[ok]] = yy[ok]
        t[todo[ok]] = tt[ok]
        todo = todo[~ok]
    nb = n - n_cl
    bx = rng.uniform(0, e, nb)
    by = rng.uniform(0, e, nb)
    bt = rng.integers(0, P, nb, endpoint=True)
    return np.concatenate([x, bx]), np.concatenate([y, by]), np.concatenate([t, bt])


def observed(cfg: Config, csr_generator=None):
    """Observed pattern of a config.  ``csr_generator(n, ring, p0, p1, seed)`` is
    the reference-exact CSR generator to use for C1/C3 (device or oracle)."""
    if cfg.kind in ("thomas", "poi"):
        x, y, t = thomas(cfg) if cfg.kind == "thomas" else poi(cfg)
        keep = inside_ring_strict(cfg, x, y)
        return x[keep], y[keep], t[keep]
    if csr_generator is None:
        raise ValueError("CSR configs need the reference-exact generator")
    return csr_generator(cfg.n, cfg.ring(), 0, cfg.period_s, cfg.seed)
