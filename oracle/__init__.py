"""Parity oracles for the space-time K pair path — TEST INFRASTRUCTURE ONLY.

Two checkers live here; neither is ever called by the product package
(``paper_1912_04753_b200``).  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module, and only as the checker or the timed CPU baseline.

* ``port``  — ``oracle/liboracle.so``, the C restatement in ``oracle/oracle.c``
  (each function cites the reference file:line it follows).
* ``ref``   — ``oracle/_ref/libstripley_ref.so``, the *unmodified* reference
  core sources (``/root/reference/proj/core/src``) compiled by
  ``oracle/Makefile`` with ``-Dstripley=stripley_ref`` plus the thin C shim
  ``oracle/ref_capi.cpp``.  Present wherever it was built (it travels to the
  GPU box as a built file); ``ref_available()`` says whether it loaded.

Arrays are numpy; surfaces are returned as ``(cs, ct)`` float64 arrays,
row-major ``[s][t]`` like the reference's ``KSurface::values``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_PORT_SO = os.path.join(_HERE, "liboracle.so")
_REF_SO = os.path.join(_HERE, "_ref", "libstripley_ref.so")
_REF_SRC = "/root/reference/proj"

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_up = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_u64 = C.c_uint64
_u32 = C.c_uint32
_i64 = C.c_int64


def build(with_ref: bool | None = None) -> None:
    """Compile the oracle(s).  The reference leg only when its sources exist."""
    subprocess.run(["make", "-s", "-C", _HERE, "all"], check=True)
    if with_ref is None:
        with_ref = os.path.isdir(_REF_SRC)
    if with_ref:
        subprocess.run(["make", "-s", "-j8", "-C", _HERE, "ref"], check=True)


_port = None
_ref = None


def _load_port():
    global _port
    if _port is None:
        if not os.path.exists(_PORT_SO):
            build(with_ref=False)
        lib = C.CDLL(_PORT_SO)
        lib.orc_pair_histogram.restype = C.c_int
        lib.orc_pair_histogram.argtypes = [
            _dp, _dp, _ip, _u64, _dp, _u32, _i64, _i64, _dp, _u32, _ip, _u32,
            _u64, _u64, C.c_int, _up, _up, _up, _dp, _up]
        lib.orc_spatial_weight.restype = C.c_double
        lib.orc_spatial_weight.argtypes = [C.c_double, C.c_double, C.c_double, _dp, _u32]
        lib.orc_temporal_weight.restype = C.c_double
        lib.orc_temporal_weight.argtypes = [_i64, _i64, _i64, _i64]
        lib.orc_point_in_polygon.restype = C.c_int
        lib.orc_point_in_polygon.argtypes = [C.c_double, C.c_double, _dp, _u32]
        lib.orc_polygon_area.restype = C.c_double
        lib.orc_polygon_area.argtypes = [_dp, _u32]
        lib.orc_finalize.restype = None
        lib.orc_finalize.argtypes = [_dp, _u64, C.c_double, _i64, _u32, _u32, _dp]
        lib.orc_to_l.restype = None
        lib.orc_to_l.argtypes = [_dp, _dp, _u32, _ip, _u32, _dp]
        lib.orc_envelopes.restype = None
        lib.orc_envelopes.argtypes = [_dp, _u32, _u32, _dp, _dp]
        lib.orc_diff.restype = None
        lib.orc_diff.argtypes = [_dp, _dp, _u32, _dp]
        lib.orc_generate_cstr.restype = None
        lib.orc_generate_cstr.argtypes = [_u64, _dp, _u32, _i64, _i64, _u64, _dp, _dp, _ip]
        for nm in ("orc_generate_bootstrap", "orc_generate_permutation"):
            f = getattr(lib, nm)
            f.restype = None
            f.argtypes = [_dp, _dp, _ip, _u64, _u64, _dp, _dp, _ip]
        lib.orc_mt_outputs.restype = None
        lib.orc_mt_outputs.argtypes = [_u64, _u64, _up]
        lib.orc_fixed_to_double.restype = C.c_double
        lib.orc_fixed_to_double.argtypes = [_u64, _u64]
        _port = lib
    return _port


def ref_available() -> bool:
    try:
        _load_ref()
        return True
    except OSError:
        return False


def _load_ref():
    global _ref
    if _ref is None:
        if not os.path.exists(_REF_SO):
            if os.path.isdir(_REF_SRC):
                build(with_ref=True)
            else:
                raise OSError("oracle/_ref/libstripley_ref.so not built and reference absent")
        lib = C.CDLL(_REF_SO)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_estimate_surface.restype = C.c_int
        lib.ref_estimate_surface.argtypes = [
            _dp, _dp, _ip, _u64, _dp, _u32, _i64, _i64, _dp, _u32, _ip, _u32,
            C.c_int, C.c_int, _dp, _up, _up]
        lib.ref_run_job.restype = C.c_int
        lib.ref_run_job.argtypes = [
            _dp, _dp, _ip, _u64, _dp, _u32, _i64, _i64, _dp, _u32, _ip, _u32,
            _u32, _u64, C.c_int, _u32, C.c_int, C.c_int, C.c_int,
            _dp, _dp, _dp, _dp, _dp, _up, _up, _dp]
        lib.ref_run_simulations.restype = C.c_int
        lib.ref_run_simulations.argtypes = [
            _dp, _dp, _ip, _u64, _dp, _u32, _i64, _i64, _dp, _u32, _ip, _u32,
            C.c_int, _u32, _u64, C.c_int, _dp]
        lib.ref_generate_cstr.restype = C.c_int
        lib.ref_generate_cstr.argtypes = [_u64, _dp, _u32, _i64, _i64, _u64, _dp, _dp, _ip]
        for nm in ("ref_generate_bootstrap", "ref_generate_permutation"):
            f = getattr(lib, nm)
            f.restype = C.c_int
            f.argtypes = [_dp, _dp, _ip, _u64, _u64, _dp, _dp, _ip]
        lib.ref_spatial_weight.restype = C.c_double
        lib.ref_spatial_weight.argtypes = [C.c_double, C.c_double, C.c_double, _dp, _u32]
        lib.ref_temporal_weight.restype = C.c_double
        lib.ref_temporal_weight.argtypes = [_i64, _i64, _i64, _i64]
        lib.ref_point_in_polygon.restype = C.c_int
        lib.ref_point_in_polygon.argtypes = [C.c_double, C.c_double, _dp, _u32]
        lib.ref_region_info.restype = C.c_int
        lib.ref_region_info.argtypes = [_dp, _u32, _i64, _i64, C.POINTER(C.c_double),
                                        C.POINTER(C.c_int64)]
        lib.ref_pair_counts.restype = C.c_int
        lib.ref_pair_counts.argtypes = [_dp, _dp, _ip, _u64, _dp, _u32, _ip, _u32, _up]
        lib.ref_pair_counts_indexed.restype = C.c_int
        lib.ref_pair_counts_indexed.argtypes = [_dp, _dp, _ip, _u64, _dp, _u32, _ip, _u32,
                                                C.c_int, _up, _up]
        lib.ref_job_open.restype = C.c_void_p
        lib.ref_job_open.argtypes = [_dp, _dp, _ip, _u64, _dp, _u32, _i64, _i64, _dp, _u32,
                                     _ip, _u32, _u64, C.c_int, _u32, C.c_int, C.c_int, C.c_int]
        lib.ref_job_pattern.restype = C.c_int
        lib.ref_job_pattern.argtypes = [C.c_void_p, _i64, _dp, _dp, _up, _up]
        lib.ref_job_close.restype = None
        lib.ref_job_close.argtypes = [C.c_void_p]
        lib.ref_brute_force_k.restype = C.c_int
        lib.ref_brute_force_k.argtypes = [_dp, _dp, _ip, _u64, _dp, _u32, _i64, _i64,
                                          _dp, _u32, _ip, _u32, _dp]
        lib.ref_regular_grid.restype = C.c_int
        lib.ref_regular_grid.argtypes = [C.c_double, C.c_double, _i64, _i64, _dp,
                                         C.POINTER(C.c_uint32), _ip, C.POINTER(C.c_uint32),
                                         _u32]
        lib.ref_random_convex_ring.restype = C.c_int
        lib.ref_random_convex_ring.argtypes = [_u64, C.c_double, C.c_double, _u32, _dp]
        lib.ref_random_star_ring.restype = C.c_int
        lib.ref_random_star_ring.argtypes = [_u64, C.c_double, _u32, _dp]
        lib.ref_uniform_points.restype = C.c_int
        lib.ref_uniform_points.argtypes = [_u64, _dp, _u32, _i64, _i64, _u64, _dp, _dp, _ip]
        lib.ref_clustered_points.restype = C.c_int
        lib.ref_clustered_points.argtypes = [_u64, _dp, _u32, _i64, _i64, _u64, _u32,
                                             C.c_double, C.c_double, _dp, _dp, _ip]
        lib.ref_mt_outputs.restype = None
        lib.ref_mt_outputs.argtypes = [_u64, _u64, _up]
        _ref = lib
    return _ref


class OracleError(ValueError):
    pass


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64a(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _ring(ring):
    r = _f64(ring).reshape(-1, 2)
    return np.ascontiguousarray(r.reshape(-1)), r.shape[0]


def _check(lib, rc):
    if rc != 0:
        raise OracleError(lib.ref_last_error().decode())


# ----------------------------------------------------------------- port (C)
class port:
    """The C restatement (oracle/oracle.c)."""

    @staticmethod
    def pair_histogram(x, y, t, ring, p0, p1, s_values, t_values, centers=None, threads=None):
        lib = _load_port()
        x, y, t = _f64(x), _f64(y), _i64a(t)
        rr, nv = _ring(ring)
        s, tv = _f64(s_values), _i64a(t_values)
        cs, ct = len(s), len(tv)
        n = len(x)
        c0, c1 = (0, n) if centers is None else centers
        counts = np.zeros(cs * ct, np.uint64)
        hi = np.zeros(cs * ct, np.uint64)
        lo = np.zeros(cs * ct, np.uint64)
        hist = np.zeros(cs * ct, np.float64)
        stats = np.zeros(4, np.uint64)
        th = threads or min(8, os.cpu_count() or 1)
        rc = lib.orc_pair_histogram(x, y, t, n, rr, nv, p0, p1, s, cs, tv, ct, c0, c1, th,
                                    counts, hi, lo, hist, stats)
        if rc != 0:
            raise OracleError("weight center outside study region")
        return dict(counts=counts.reshape(cs, ct), sum_hi=hi.reshape(cs, ct),
                    sum_lo=lo.reshape(cs, ct), hist=hist.reshape(cs, ct),
                    in_threshold=int(stats[0]), arc_pairs=int(stats[1]),
                    half_pairs=int(stats[2]))

    @staticmethod
    def finalize(hist, n, area, duration):
        lib = _load_port()
        h = _f64(hist)
        cs, ct = h.shape
        k = np.zeros((cs, ct), np.float64)
        lib.orc_finalize(np.ascontiguousarray(h.reshape(-1)), n, area, duration, cs, ct, k.reshape(-1))
        return k

    @staticmethod
    def to_l(k, s_values, t_values):
        lib = _load_port()
        k = _f64(k)
        cs, ct = k.shape
        out = np.zeros_like(k)
        lib.orc_to_l(np.ascontiguousarray(k.reshape(-1)), _f64(s_values), cs, _i64a(t_values), ct,
                     out.reshape(-1))
        return out

    @staticmethod
    def envelopes(l_all):
        lib = _load_port()
        la = _f64(l_all)
        m, cs, ct = la.shape
        up = np.zeros((cs, ct)); lo = np.zeros((cs, ct))
        lib.orc_envelopes(np.ascontiguousarray(la.reshape(-1)), m, cs * ct, up.reshape(-1), lo.reshape(-1))
        return up, lo

    @staticmethod
    def diff(est_l, upper):
        lib = _load_port()
        e, u = _f64(est_l), _f64(upper)
        out = np.zeros_like(e)
        lib.orc_diff(np.ascontiguousarray(e.reshape(-1)), np.ascontiguousarray(u.reshape(-1)),
                     e.size, out.reshape(-1))
        return out

    @staticmethod
    def area(ring):
        rr, nv = _ring(ring)
        return _load_port().orc_polygon_area(rr, nv)

    @staticmethod
    def spatial_weight(cx, cy, d, ring):
        rr, nv = _ring(ring)
        return _load_port().orc_spatial_weight(cx, cy, d, rr, nv)

    @staticmethod
    def temporal_weight(ct, u, p0, p1):
        return _load_port().orc_temporal_weight(ct, u, p0, p1)

    @staticmethod
    def point_in_polygon(px, py, ring):
        rr, nv = _ring(ring)
        return bool(_load_port().orc_point_in_polygon(px, py, rr, nv))

    @staticmethod
    def generate_cstr(n, ring, p0, p1, seed):
        rr, nv = _ring(ring)
        x = np.zeros(n); y = np.zeros(n); t = np.zeros(n, np.int64)
        _load_port().orc_generate_cstr(n, rr, nv, p0, p1, seed, x, y, t)
        return x, y, t

    @staticmethod
    def generate_bootstrap(x, y, t, seed):
        n = len(x)
        ox = np.zeros(n); oy = np.zeros(n); ot = np.zeros(n, np.int64)
        _load_port().orc_generate_bootstrap(_f64(x), _f64(y), _i64a(t), n, seed, ox, oy, ot)
        return ox, oy, ot

    @staticmethod
    def generate_permutation(x, y, t, seed):
        n = len(x)
        ox = np.zeros(n); oy = np.zeros(n); ot = np.zeros(n, np.int64)
        _load_port().orc_generate_permutation(_f64(x), _f64(y), _i64a(t), n, seed, ox, oy, ot)
        return ox, oy, ot

    @staticmethod
    def mt_outputs(seed, count):
        out = np.zeros(count, np.uint64)
        _load_port().orc_mt_outputs(seed, count, out)
        return out

    @staticmethod
    def estimate(x, y, t, ring, p0, p1, s_values, t_values, threads=None):
        """K, L, counts and exact hist for one pattern (port path end to end)."""
        h = port.pair_histogram(x, y, t, ring, p0, p1, s_values, t_values, threads=threads)
        k = port.finalize(h["hist"], len(x), port.area(ring), p1 - p0)
        h["k"] = k
        h["l"] = port.to_l(k, s_values, t_values)
        return h


# ----------------------------------------------------------- ref (C++ ref)
class ref:
    """The reference itself, compiled from /root/reference/proj/core/src."""

    @staticmethod
    def estimate_surface(x, y, t, ring, p0, p1, s_values, t_values, use_index=True,
                         use_cache=False):
        lib = _load_ref()
        rr, nv = _ring(ring)
        s, tv = _f64(s_values), _i64a(t_values)
        out = np.zeros(len(s) * len(tv))
        pairs = np.zeros(1, np.uint64); comps = np.zeros(1, np.uint64)
        _check(lib, lib.ref_estimate_surface(_f64(x), _f64(y), _i64a(t), len(x), rr, nv, p0, p1,
                                             s, len(s), tv, len(tv), int(use_index),
                                             int(use_cache), out, pairs, comps))
        return out.reshape(len(s), len(tv)), int(pairs[0]), int(comps[0])

    @staticmethod
    def run_job(x, y, t, ring, p0, p1, s_values, t_values, sims, seed, method=0,
                partitions=1, workers=1, use_index=True, use_cache=False):
        lib = _load_ref()
        rr, nv = _ring(ring)
        s, tv = _f64(s_values), _i64a(t_values)
        b = len(s) * len(tv)
        outs = [np.zeros(b) for _ in range(5)]
        pairs = np.zeros(1, np.uint64); comps = np.zeros(1, np.uint64)
        secs = np.zeros(3)
        _check(lib, lib.ref_run_job(_f64(x), _f64(y), _i64a(t), len(x), rr, nv, p0, p1, s, len(s),
                                    tv, len(tv), sims, seed, method, partitions, workers,
                                    int(use_index), int(use_cache), *outs, pairs, comps, secs))
        shp = (len(s), len(tv))
        res = dict(k=outs[0].reshape(shp), l=outs[1].reshape(shp), in_threshold=int(pairs[0]),
                   comparisons=int(comps[0]), seconds=secs.copy())
        if sims > 0:
            res.update(upper=outs[2].reshape(shp), lower=outs[3].reshape(shp),
                       diff=outs[4].reshape(shp))
        return res

    @staticmethod
    def run_simulations(x, y, t, ring, p0, p1, s_values, t_values, m, base_seed, method=0,
                        use_index=True):
        lib = _load_ref()
        rr, nv = _ring(ring)
        s, tv = _f64(s_values), _i64a(t_values)
        out = np.zeros(m * len(s) * len(tv))
        _check(lib, lib.ref_run_simulations(_f64(x), _f64(y), _i64a(t), len(x), rr, nv, p0, p1,
                                            s, len(s), tv, len(tv), method, m, base_seed,
                                            int(use_index), out))
        return out.reshape(m, len(s), len(tv))

    @staticmethod
    def generate_cstr(n, ring, p0, p1, seed):
        lib = _load_ref()
        rr, nv = _ring(ring)
        x = np.zeros(n); y = np.zeros(n); t = np.zeros(n, np.int64)
        _check(lib, lib.ref_generate_cstr(n, rr, nv, p0, p1, seed, x, y, t))
        return x, y, t

    @staticmethod
    def generate_bootstrap(x, y, t, seed):
        lib = _load_ref()
        n = len(x)
        ox = np.zeros(n); oy = np.zeros(n); ot = np.zeros(n, np.int64)
        _check(lib, lib.ref_generate_bootstrap(_f64(x), _f64(y), _i64a(t), n, seed, ox, oy, ot))
        return ox, oy, ot

    @staticmethod
    def generate_permutation(x, y, t, seed):
        lib = _load_ref()
        n = len(x)
        ox = np.zeros(n); oy = np.zeros(n); ot = np.zeros(n, np.int64)
        _check(lib, lib.ref_generate_permutation(_f64(x), _f64(y), _i64a(t), n, seed, ox, oy, ot))
        return ox, oy, ot

    @staticmethod
    def spatial_weight(cx, cy, d, ring):
        rr, nv = _ring(ring)
        return _load_ref().ref_spatial_weight(cx, cy, d, rr, nv)

    @staticmethod
    def temporal_weight(ct, u, p0, p1):
        return _load_ref().ref_temporal_weight(ct, u, p0, p1)

    @staticmethod
    def point_in_polygon(px, py, ring):
        rr, nv = _ring(ring)
        return bool(_load_ref().ref_point_in_polygon(px, py, rr, nv))

    @staticmethod
    def region_info(ring, p0, p1):
        lib = _load_ref()
        rr, nv = _ring(ring)
        a = C.c_double(); d = C.c_int64()
        _check(lib, lib.ref_region_info(rr, nv, p0, p1, C.byref(a), C.byref(d)))
        return a.value, d.value

    @staticmethod
    def pair_counts(x, y, t, s_values, t_values):
        lib = _load_ref()
        s, tv = _f64(s_values), _i64a(t_values)
        out = np.zeros(len(s) * len(tv), np.uint64)
        _check(lib, lib.ref_pair_counts(_f64(x), _f64(y), _i64a(t), len(x), s, len(s), tv,
                                        len(tv), out))
        return out.reshape(len(s), len(tv))

    @staticmethod
    def pair_counts_indexed(x, y, t, s_values, t_values, threads=0):
        """Per-bin counts over the reference's STR R-tree (threaded)."""
        lib = _load_ref()
        s, tv = _f64(s_values), _i64a(t_values)
        out = np.zeros(len(s) * len(tv), np.uint64)
        tot = np.zeros(1, np.uint64)
        _check(lib, lib.ref_pair_counts_indexed(_f64(x), _f64(y), _i64a(t), len(x), s, len(s),
                                                tv, len(tv), int(threads), out, tot))
        return out.reshape(len(s), len(tv))

    class Job:
        """rt::run_job split per pattern (ref_job_open / ref_job_pattern): plan once on
        the observed points, then run the observed pattern (``pattern(-1)``) or
        realisation r (``pattern(r)``: sim::generate with seed + r) through the
        reference's make_tasks -> LocalExecutor::run -> aggregate -> to_l."""

        def __init__(self, x, y, t, ring, p0, p1, s_values, t_values, seed, method=0,
                     partitions=1, workers=0, use_index=True, use_cache=False):
            lib = _load_ref()
            rr, nv = _ring(ring)
            self._s, self._tv = _f64(s_values), _i64a(t_values)
            self._keep = (_f64(x), _f64(y), _i64a(t), rr)
            self._h = lib.ref_job_open(self._keep[0], self._keep[1], self._keep[2], len(x), rr,
                                       nv, p0, p1, self._s, len(self._s), self._tv,
                                       len(self._tv), seed, method, partitions, int(workers),
                                       int(use_index), int(use_cache))
            if not self._h:
                raise OracleError(lib.ref_last_error().decode())

        def pattern(self, which):
            lib = _load_ref()
            shp = (len(self._s), len(self._tv))
            k = np.zeros(shp); l = np.zeros(shp)
            pairs = np.zeros(1, np.uint64); comps = np.zeros(1, np.uint64)
            _check(lib, lib.ref_job_pattern(self._h, int(which), k.reshape(-1), l.reshape(-1),
                                            pairs, comps))
            return dict(k=k, l=l, in_threshold=int(pairs[0]), comparisons=int(comps[0]))

        def close(self):
            if self._h:
                _load_ref().ref_job_close(self._h)
                self._h = None

        def __del__(self):
            try:
                self.close()
            except Exception:
                pass

    @staticmethod
    def brute_force_k(x, y, t, ring, p0, p1, s_values, t_values):
        lib = _load_ref()
        rr, nv = _ring(ring)
        s, tv = _f64(s_values), _i64a(t_values)
        out = np.zeros(len(s) * len(tv))
        _check(lib, lib.ref_brute_force_k(_f64(x), _f64(y), _i64a(t), len(x), rr, nv, p0, p1, s,
                                          len(s), tv, len(tv), out))
        return out.reshape(len(s), len(tv))

    @staticmethod
    def regular_grid(s_step, s_max, t_step, t_max):
        lib = _load_ref()
        cap = 100000
        s = np.zeros(cap); tv = np.zeros(cap, np.int64)
        cs = C.c_uint32(); ct = C.c_uint32()
        _check(lib, lib.ref_regular_grid(s_step, s_max, t_step, t_max, s, C.byref(cs), tv,
                                         C.byref(ct), cap))
        return s[: cs.value].copy(), tv[: ct.value].copy()

    @staticmethod
    def random_convex_ring(seed, rx, ry, vertices):
        out = np.zeros(2 * vertices)
        _check(_load_ref(), _load_ref().ref_random_convex_ring(seed, rx, ry, vertices, out))
        return out.reshape(-1, 2)

    @staticmethod
    def random_star_ring(seed, radius, vertices):
        out = np.zeros(2 * vertices)
        _check(_load_ref(), _load_ref().ref_random_star_ring(seed, radius, vertices, out))
        return out.reshape(-1, 2)

    @staticmethod
    def uniform_points(seed, ring, p0, p1, n):
        lib = _load_ref()
        rr, nv = _ring(ring)
        x = np.zeros(n); y = np.zeros(n); t = np.zeros(n, np.int64)
        _check(lib, lib.ref_uniform_points(seed, rr, nv, p0, p1, n, x, y, t))
        return x, y, t

    @staticmethod
    def clustered_points(seed, ring, p0, p1, n, clusters, sigma_s, sigma_t):
        lib = _load_ref()
        rr, nv = _ring(ring)
        x = np.zeros(n); y = np.zeros(n); t = np.zeros(n, np.int64)
        _check(lib, lib.ref_clustered_points(seed, rr, nv, p0, p1, n, clusters, sigma_s, sigma_t,
                                             x, y, t))
        return x, y, t

    @staticmethod
    def mt_outputs(seed, count):
        out = np.zeros(count, np.uint64)
        _load_ref().ref_mt_outputs(seed, count, out)
        return out
