"""``stripley::sim`` mirror (proj/core/include/stripley/simulation.hpp).

Realisations are generated on the device with a bit-exact MT19937-64
(the reference's ``rng::Engine``), so realisation r of seed ladder
``base_seed + r`` is the reference's point pattern, bit for bit.
"""
from __future__ import annotations

import ctypes as C
from enum import IntEnum

import numpy as np

from .. import _lib
from . import device as _device
from .est import (DistanceGrid, EstimatorOptions, EstimatorTelemetry, KSurface, SurfaceKind,
                  _prepare)
from .geom import Points, StudyRegion


class Method(IntEnum):  # simulation.hpp:14
    Cstr = _lib.METHOD_CSR
    Bootstrap = _lib.METHOD_BOOTSTRAP
    Permutation = _lib.METHOD_PERMUTATION


def generate_cstr(n: int, region: StudyRegion, seed: int, device=None) -> Points:
    """``sim::generate_cstr`` (simulation.cpp:10-24), generated on the device."""
    d = device if isinstance(device, _device.Device) else _device.get(device)
    d.configure(region)
    x = np.zeros(n)
    y = np.zeros(n)
    t = np.zeros(n, np.int64)
    d.check(d.lib.stk_generate_cstr(d.h, int(n), int(seed), _lib.ptr(x), _lib.ptr(y),
                                    _lib.ptr(t, C.c_int64)))
    return Points(x, y, t)


def simulate(points, region: StudyRegion, grid: DistanceGrid, method: Method, r_begin: int,
             r_end: int, base_seed: int, keep_surfaces: bool = True, device=None,
             telemetry: EstimatorTelemetry | None = None):
    """Realisations ``r`` in ``[r_begin, r_end)``: their L surfaces (if
    ``keep_surfaces``) and the pointwise max/min over them."""
    pts, d = _prepare(points, region, grid, None, device)
    m = max(0, r_end - r_begin)
    shape = (grid.cells_s(), grid.cells_t())
    l_all = np.zeros((m,) + shape) if keep_surfaces else None
    up = np.zeros(shape)
    lo = np.zeros(shape)
    tel = _lib.StkTelemetry()
    needs_obs = Method(method) != Method.Cstr
    d.check(d.lib.stk_simulate(
        d.h, _lib.ptr(pts.x) if needs_obs else None, _lib.ptr(pts.y) if needs_obs else None,
        _lib.ptr(pts.t, C.c_int64) if needs_obs else None, len(pts), int(method),
        int(base_seed), int(r_begin), int(r_end), _lib.ptr(l_all) if keep_surfaces else None,
        _lib.ptr(up), _lib.ptr(lo), C.byref(tel)))
    if telemetry is not None:
        telemetry.add(tel)
    return l_all, up, lo


def run_simulations(points, region: StudyRegion, grid: DistanceGrid, method: Method, m: int,
                    base_seed: int, options: EstimatorOptions | None = None,
                    weight_cache=None, device=None) -> list[KSurface]:
    """``sim::run_simulations`` (simulation.cpp:67-84): m L surfaces."""
    if m < 1:
        raise ValueError("need at least one simulation")
    if weight_cache is not None:
        weight_cache.freeze()
    l_all, _, _ = simulate(points, region, grid, method, 0, m, base_seed, True, device)
    return [KSurface(grid, l_all[r], SurfaceKind.L) for r in range(m)]


def envelopes(sims) -> tuple[KSurface, KSurface]:
    """``sim::envelopes`` (simulation.cpp:86-102): pointwise max/min."""
    sims = list(sims)
    if not sims:
        raise ValueError("envelopes need >= 1 surface")
    for s in sims:
        if s.grid != sims[0].grid:
            raise ValueError("grid mismatch between simulated surfaces")
    up = np.array(sims[0].values, copy=True)
    lo = np.array(sims[0].values, copy=True)
    for s in sims[1:]:
        v = s.values
        up = np.where(up < v, v, up)
        lo = np.where(v < lo, v, lo)
    return KSurface(sims[0].grid, up, sims[0].kind), KSurface(sims[0].grid, lo, sims[0].kind)
