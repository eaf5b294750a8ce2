"""``stripley::geom`` mirror (proj/core/include/stripley/geometry.hpp).

Points travel as structure-of-arrays (``Points``: x, y float64; t int64), the
layout the device kernels read; ``STPoint``/``make_point`` keep the reference's
record form for small inputs.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from enum import IntEnum

import numpy as np

from .. import _lib


class TimeUnit(IntEnum):  # geometry.hpp:9-15
    Seconds = 0
    Minutes = 1
    Hours = 2
    Days = 3
    Months = 4


@dataclass
class STPoint:  # geometry.hpp:20-29
    x: float = 0.0
    y: float = 0.0
    overlap_count: int = 1
    start_time: int = 0
    end_time: int = 0
    zone_id: int = 0


def make_point(x: float, y: float, t: int) -> STPoint:  # geometry.hpp:31-33
    return STPoint(float(x), float(y), 1, int(t), int(t), 0)


class Points:
    """A point pattern as SoA: ``x``, ``y`` (float64) and ``t`` (int64 start_time)."""

    __slots__ = ("x", "y", "t")

    def __init__(self, x, y, t):
        self.x = _lib.f64(x)
        self.y = _lib.f64(y)
        self.t = _lib.i64(t)
        if not (len(self.x) == len(self.y) == len(self.t)):
            raise ValueError("x, y, t lengths differ")

    @staticmethod
    def of(points) -> "Points":
        """Accept Points, an (x, y, t) tuple, or a sequence of STPoint."""
        if isinstance(points, Points):
            return points
        if isinstance(points, tuple) and len(points) == 3:
            return Points(*points)
        pts = list(points)
        return Points([p.x for p in pts], [p.y for p in pts], [p.start_time for p in pts])

    def __len__(self):
        return len(self.x)

    def __getitem__(self, i) -> STPoint:
        return make_point(self.x[i], self.y[i], self.t[i])


@dataclass
class STEnvelope:  # geometry.hpp:36-58
    x_min: float = 0.0
    x_max: float = 0.0
    y_min: float = 0.0
    y_max: float = 0.0
    t_min: int = 0
    t_max: int = 0


class StudyRegion:
    """``geom::StudyRegion`` (geometry.hpp:95-120): simple polygon + period.

    Validation runs in libstk's context-free ``stk_check_region`` with the
    reference's checks and messages (geometry.cpp:110-136); closed rings are
    accepted and stored open.
    """

    def __init__(self, ring, period_start: int, period_end: int):
        r = _lib.f64(np.asarray(ring, dtype=np.float64).reshape(-1, 2).reshape(-1))
        lib = _lib.load()
        area = C.c_double()
        dur = C.c_int64()
        msg = C.create_string_buffer(256)
        rc = lib.stk_check_region(_lib.ptr(r), len(r) // 2, int(period_start), int(period_end),
                                  C.byref(area), C.byref(dur), msg, 256)
        if rc != 0:
            raise ValueError(msg.value.decode())
        ring2 = r.reshape(-1, 2)
        if len(ring2) >= 2 and ring2[0, 0] == ring2[-1, 0] and ring2[0, 1] == ring2[-1, 1]:
            ring2 = ring2[:-1]
        self._ring = np.ascontiguousarray(ring2)
        self._p0 = int(period_start)
        self._p1 = int(period_end)
        self._area = area.value
        self._duration = dur.value

    def boundary(self) -> np.ndarray:
        return self._ring

    def period_start(self) -> int:
        return self._p0

    def period_end(self) -> int:
        return self._p1

    def area(self) -> float:
        return self._area

    def duration(self) -> int:
        return self._duration

    def bounding_envelope(self) -> STEnvelope:  # geometry.cpp:138-153
        r = self._ring
        return STEnvelope(float(r[:, 0].min()), float(r[:, 0].max()), float(r[:, 1].min()),
                          float(r[:, 1].max()), self._p0, self._p1)

    def key(self):
        return (self._ring.tobytes(), self._p0, self._p1)

    def __eq__(self, other):
        return isinstance(other, StudyRegion) and self.key() == other.key()

    def __hash__(self):
        return hash(self.key())


def rectangle(x0: float, y0: float, x1: float, y1: float, period_start: int,
              period_end: int) -> StudyRegion:
    """Axis-aligned rectangular study region (the configs' regions)."""
    return StudyRegion([[x0, y0], [x1, y0], [x1, y1], [x0, y1]], period_start, period_end)
