"""``stripley::est`` mirror (proj/core/include/stripley/estimator.hpp).

``estimate_surface`` runs entirely on the device (grid build, pair kernel,
finalize) through ``stk_estimate_surface``.  The small surface utilities
(``to_l``, ``theoretical_surface``, ``diff_surface``, ``bin_pair``) act on host
surfaces the caller already holds, exactly like the reference's.
"""
from __future__ import annotations

import bisect
import ctypes as C
import math
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from .. import _lib
from . import device as _device
from .geom import Points, StudyRegion

PI = 3.14159265358979323846


class DistanceGrid:
    """``est::DistanceGrid`` (estimator.hpp:15-29): ascending positive thresholds."""

    def __init__(self, s_values, t_values):
        self.s_values = [float(v) for v in s_values]
        self.t_values = [int(v) for v in t_values]

    def validate(self):  # estimator.cpp:14-22 via the library's own check
        s = _lib.f64(self.s_values)
        t = _lib.i64(self.t_values)
        msg = C.create_string_buffer(256)
        rc = _lib.load().stk_check_grid(_lib.ptr(s), len(s), _lib.ptr(t, C.c_int64), len(t), msg,
                                        256)
        if rc != 0:
            raise ValueError(msg.value.decode())

    def s_max(self) -> float:
        return self.s_values[-1]

    def t_max(self) -> int:
        return self.t_values[-1]

    def cells_s(self) -> int:
        return len(self.s_values)

    def cells_t(self) -> int:
        return len(self.t_values)

    @staticmethod
    def regular(s_step: float, s_max: float, t_step: int, t_max: int) -> "DistanceGrid":
        """estimator.cpp:24-32 — note the accumulating ``s += s_step``."""
        s_vals = []
        s = float(s_step)
        while s <= s_max * (1.0 + 1e-12):
            s_vals.append(s)
            s += s_step
        t_vals = list(range(int(t_step), int(t_max) + 1, int(t_step))) if t_step > 0 else []
        g = DistanceGrid(s_vals, t_vals)
        g.validate()
        return g

    def key(self):
        return (tuple(self.s_values), tuple(self.t_values))

    def __eq__(self, other):
        return isinstance(other, DistanceGrid) and self.key() == other.key()

    def __hash__(self):
        return hash(self.key())


class SurfaceKind(Enum):
    K = 0
    L = 1
    Diff = 2


@dataclass
class KSurface:
    """``est::KSurface``: ``values[si][ti]`` as a (cells_s, cells_t) float64 array."""

    grid: DistanceGrid
    values: np.ndarray
    kind: SurfaceKind = SurfaceKind.K


@dataclass
class EstimatorOptions:  # estimator.hpp:39-45
    use_index: bool = False
    use_cache: bool = False
    coord_tolerance: float = 0.0
    dist_tolerance: float = 0.0
    node_capacity: int = 16


@dataclass
class EstimatorTelemetry:  # estimator.hpp:47-51 (+ device counters)
    pair_comparisons: int = 0
    in_threshold_pairs: int = 0
    index_build_seconds: float = 0.0
    exact_path_pairs: int = 0
    device: dict = field(default_factory=dict)

    def add(self, t: "_lib.StkTelemetry"):
        self.pair_comparisons += int(t.candidate_pairs)
        self.in_threshold_pairs += int(t.in_threshold_pairs)
        self.index_build_seconds += float(t.grid_ms) * 1e-3
        self.exact_path_pairs += int(t.exact_path_pairs)
        for k, v in t.as_dict().items():
            self.device[k] = self.device.get(k, 0) + v


class WeightCache:
    """``cache::WeightCache`` stand-in.  At tolerance 0 the reference cache never
    changes results (tests/test_estimator.cpp:130-151); the device recomputes
    weights per center instead.  Nonzero tolerances are order-dependent in the
    reference and are rejected."""

    def __init__(self, coord_tolerance: float = 0.0, dist_tolerance: float = 0.0):
        self.coord_tolerance = coord_tolerance
        self.dist_tolerance = dist_tolerance
        self.frozen = False

    def freeze(self):
        self.frozen = True


def intensity(n: int, region: StudyRegion) -> float:  # estimator.cpp:45-49
    if n == 0:
        raise ValueError("intensity needs n >= 1")
    return float(n) / (region.area() * float(region.duration()))


def theoretical_k(s: float, t: float) -> float:  # estimator.cpp:51
    return 2.0 * PI * s * s * t


def k_to_l(k: float, s: float, t: float) -> float:  # estimator.cpp:53-57
    if t == 0.0:
        raise ValueError("L transform undefined at t=0")
    if k < 0.0:
        raise ValueError("K value must be >= 0")
    return math.sqrt(k / (2.0 * PI * t)) - s


def theoretical_surface(grid: DistanceGrid) -> KSurface:  # estimator.cpp:59-69
    v = np.zeros((grid.cells_s(), grid.cells_t()))
    for si, s in enumerate(grid.s_values):
        for ti, t in enumerate(grid.t_values):
            v[si, ti] = theoretical_k(s, float(t))
    return KSurface(grid, v, SurfaceKind.K)


def to_l(k_surface: KSurface) -> KSurface:  # estimator.cpp:71-82
    g = k_surface.grid
    v = np.array(k_surface.values, dtype=np.float64, copy=True)
    for si, s in enumerate(g.s_values):
        for ti, t in enumerate(g.t_values):
            v[si, ti] = k_to_l(float(k_surface.values[si, ti]), s, float(t))
    return KSurface(g, v, SurfaceKind.L)


def bin_pair(grid: DistanceGrid, d: float, u: int):  # estimator.cpp:84-92
    si = bisect.bisect_left(grid.s_values, d)
    if si == len(grid.s_values):
        return None
    ti = bisect.bisect_left(grid.t_values, u)
    if ti == len(grid.t_values):
        return None
    return si, ti


def diff_surface(estimated_l: KSurface, upper_l: KSurface) -> KSurface:  # estimator.cpp:188-202
    if estimated_l.grid != upper_l.grid:
        raise ValueError("grid mismatch between surfaces")
    e, u = estimated_l.values, upper_l.values
    return KSurface(estimated_l.grid, np.where(e > u, e - u, 0.0), SurfaceKind.Diff)


def _prepare(points, region: StudyRegion, grid: DistanceGrid, options, dev):
    grid.validate()
    pts = Points.of(points)
    if len(pts) < 2:
        raise ValueError("K estimation needs n >= 2")
    d = dev if isinstance(dev, _device.Device) else _device.get(dev)
    d.configure(region, grid, options)
    return pts, d


def estimate_surface(points, region: StudyRegion, grid: DistanceGrid,
                     options: EstimatorOptions | None = None, weight_cache=None,
                     telemetry: EstimatorTelemetry | None = None, device=None) -> KSurface:
    """``est::estimate_surface`` (estimator.hpp:107-111) on the device."""
    options = options or EstimatorOptions()
    if weight_cache is not None and options.use_cache and (
            weight_cache.coord_tolerance or weight_cache.dist_tolerance):
        raise NotImplementedError("nonzero weight-cache tolerances are not supported")
    pts, d = _prepare(points, region, grid, options, device)
    k = np.zeros((grid.cells_s(), grid.cells_t()))
    tel = _lib.StkTelemetry()
    d.check(d.lib.stk_estimate_surface(d.h, _lib.ptr(pts.x), _lib.ptr(pts.y),
                                       _lib.ptr(pts.t, C.c_int64), len(pts), _lib.ptr(k),
                                       C.byref(tel)))
    if telemetry is not None:
        telemetry.add(tel)
    return KSurface(grid, k, SurfaceKind.K)


def pair_histogram(points, region: StudyRegion, grid: DistanceGrid, shard: int = 0,
                   nshards: int = 1, device=None, telemetry: EstimatorTelemetry | None = None):
    """Pre-cumulative per-bin results of one pattern (or one shard of it):
    exact ``counts`` (uint64), the exact weighted sum as 128-bit fixed point
    (``sum_hi``, ``sum_lo``; 53 fractional bits) and ``hist`` (that sum rounded
    once) — est::PairHistogram (estimator.hpp:55-81)."""
    pts, d = _prepare(points, region, grid, None, device)
    shape = (grid.cells_s(), grid.cells_t())
    counts = np.zeros(shape, np.uint64)
    hi = np.zeros(shape, np.uint64)
    lo = np.zeros(shape, np.uint64)
    hist = np.zeros(shape, np.float64)
    tel = _lib.StkTelemetry()
    d.check(d.lib.stk_pair_histogram(d.h, _lib.ptr(pts.x), _lib.ptr(pts.y),
                                     _lib.ptr(pts.t, C.c_int64), len(pts), int(shard),
                                     int(nshards), _lib.ptr(counts, C.c_uint64),
                                     _lib.ptr(hi, C.c_uint64), _lib.ptr(lo, C.c_uint64),
                                     _lib.ptr(hist), C.byref(tel)))
    if telemetry is not None:
        telemetry.add(tel)
    return dict(counts=counts, sum_hi=hi, sum_lo=lo, hist=hist,
                in_threshold=int(tel.in_threshold_pairs), exact_path=int(tel.exact_path_pairs),
                telemetry=tel)


def finalize_exact(sum_hi, sum_lo, n: int, region: StudyRegion, grid: DistanceGrid,
                   device=None):
    """est::finalize_surface + to_l from exact 128-bit sums (reference order)."""
    d = device if isinstance(device, _device.Device) else _device.get(device)
    d.configure(region, grid)
    hi = np.ascontiguousarray(sum_hi, dtype=np.uint64)
    lo = np.ascontiguousarray(sum_lo, dtype=np.uint64)
    k = np.zeros(hi.shape)
    l = np.zeros(hi.shape)
    d.check(d.lib.stk_finalize(d.h, int(n), _lib.ptr(hi, C.c_uint64), _lib.ptr(lo, C.c_uint64),
                               _lib.ptr(k), _lib.ptr(l)))
    return KSurface(grid, k, SurfaceKind.K), KSurface(grid, l, SurfaceKind.L)
