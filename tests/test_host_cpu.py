"""CPU: the C ABI library and the host-side mirror of the reference API.

No compute calls here (no GPU): libstk.so loads, exports every symbol that
include/stk.h declares, validates regions and grids with the reference's
rules and messages, and the host mirror's utilities match the reference.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle
from conftest import ROOT, golden

from paper_1912_04753_b200 import _lib
from paper_1912_04753_b200.stripley import est, geom, rt, sim


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "stk.h")).read()
    return sorted(set(re.findall(r"\b(stk_[a-z0-9_]+)\s*\(", hdr)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_symbols()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    assert sorted(_lib.EXPORTED) == names


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_version_string():
    assert b"sm_100a" in _lib.load().stk_version()


REGION_CASES = [
    ([[0, 0], [10, 0], [10, 10], [0, 10]], 0, 100, None),
    ([[0, 0], [10, 0], [10, 10], [0, 10], [0, 0]], 0, 100, None),  # closed ring accepted
    ([[0, 0], [10, 0]], 0, 100, "polygon needs >= 3 vertices"),
    ([[0, 0], [10, 0], [np.nan, 10]], 0, 100, "polygon vertex not finite"),
    ([[0, 0], [10, 10], [10, 0], [0, 10]], 0, 100, "polygon is self-intersecting"),
    ([[0, 0], [1, 1], [2, 2]], 0, 100, "degenerate polygon (zero area)"),
    ([[0, 0], [10, 0], [10, 10]], 5, 5, "study period duration must be > 0"),
]


@pytest.mark.parametrize("ring,p0,p1,msg", REGION_CASES)
def test_region_validation_matches_reference(ring, p0, p1, msg):
    if msg is None:
        r = geom.StudyRegion(ring, p0, p1)
        assert r.area() == 100.0 and r.duration() == p1 - p0 and len(r.boundary()) == 4
    else:
        with pytest.raises(ValueError, match=re.escape(msg)):
            geom.StudyRegion(ring, p0, p1)
    if oracle.ref_available():
        from oracle import ref

        try:
            ref.region_info(np.array(ring, float), p0, p1)
            ref_msg = None
        except oracle.OracleError as e:
            ref_msg = str(e)
        assert ref_msg == msg


GRID_CASES = [
    ([0.0, 1.0], [1], "distance grid must exclude s=0 and t=0"),
    ([1.0, 1.0], [1], "distance grid must be strictly increasing"),
    ([2.0, 1.0], [1], "distance grid must be strictly increasing"),
    ([1.0], [0], "distance grid must exclude s=0 and t=0"),
    ([], [1], "distance grid must be non-empty"),
    ([1.0, 2.0], [1, 2], None),
]


@pytest.mark.parametrize("s,t,msg", GRID_CASES)
def test_grid_validation_matches_reference(s, t, msg):
    """proj/tests/test_estimator.cpp:17-30."""
    g = est.DistanceGrid(s, t)
    if msg is None:
        g.validate()
    else:
        with pytest.raises(ValueError, match=re.escape(msg)):
            g.validate()


def test_regular_grid_matches_reference():
    g = est.DistanceGrid.regular(500.0, 2000.0, 2, 10)
    assert g.s_values == [500, 1000, 1500, 2000] and g.t_values == [2, 4, 6, 8, 10]
    if oracle.ref_available():
        from oracle import ref

        for args in [(100, 2000, 5, 100), (93.75, 1500, 540000, 8640000), (0.1, 1.0, 1, 3),
                     (50, 1000, 129600, 2592000)]:
            s, t = ref.regular_grid(*args)
            g = est.DistanceGrid.regular(*args)
            assert g.s_values == list(s) and g.t_values == list(t)


def test_bin_pair_semantics():
    """proj/tests/test_estimator.cpp:52-60."""
    g = est.DistanceGrid([1.0, 2.0, 3.0], [10, 20])
    assert est.bin_pair(g, 0.5, 5) == (0, 0)
    assert est.bin_pair(g, 1.0, 10) == (0, 0)
    assert est.bin_pair(g, 1.5, 11) == (1, 1)
    assert est.bin_pair(g, 3.0, 20) == (2, 1)
    assert est.bin_pair(g, 3.1, 5) is None
    assert est.bin_pair(g, 1.0, 21) is None


def test_theoretical_and_l_transform():
    """proj/tests/test_estimator.cpp:32-50."""
    assert est.theoretical_k(1.0, 1.0) == pytest.approx(2 * np.pi)
    for s in (0.5, 10.0, 3000.0):
        for t in (1.0, 7.0, 50.0):
            assert est.k_to_l(est.theoretical_k(s, t), s, t) == pytest.approx(0.0, abs=1e-9)
    with pytest.raises(ValueError):
        est.k_to_l(1.0, 1.0, 0.0)
    with pytest.raises(ValueError):
        est.k_to_l(-1.0, 1.0, 1.0)
    g = est.DistanceGrid.regular(1.0, 3.0, 1, 2)
    theo = est.theoretical_surface(g)
    assert theo.values[1, 0] == pytest.approx(2 * np.pi * 4)
    assert np.allclose(est.to_l(theo).values, 0.0, atol=1e-12)


def test_diff_and_envelopes():
    g = est.DistanceGrid([1.0, 2.0], [1])
    d = est.diff_surface(est.KSurface(g, np.array([[3.0], [-1.0]]), est.SurfaceKind.L),
                         est.KSurface(g, np.array([[2.0], [0.5]]), est.SurfaceKind.L))
    assert d.kind == est.SurfaceKind.Diff and d.values[0, 0] == 1.0 and d.values[1, 0] == 0.0
    sims = [est.KSurface(g, np.array([[v], [-v]]), est.SurfaceKind.L) for v in (1.0, 3.0, 2.0)]
    up, lo = sim.envelopes(sims)
    assert up.values[0, 0] == 3.0 and lo.values[1, 0] == -3.0
    with pytest.raises(ValueError, match="envelopes need >= 1 surface"):
        sim.envelopes([])
    with pytest.raises(ValueError, match="grid mismatch"):
        sim.envelopes([sims[0], est.KSurface(est.DistanceGrid([1.0], [1]), np.zeros((1, 1)))])


def test_shard_ranges_partition():
    for total in (0, 1, 7, 99, 199):
        for world in (1, 2, 3, 8):
            rs = [rt.shard_range(total, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == total
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1


def test_limbs_roundtrip_exact():
    """pack_limbs / unpack_limbs (the algebra of the device's pack/unpack
    kernels): summing limbs of W partials equals the 128-bit sum mod 2^128."""
    rng = np.random.default_rng(3)
    hi = rng.integers(0, 2**40, 50, dtype=np.uint64)
    lo = rng.integers(0, 2**63, 50, dtype=np.uint64) * np.uint64(2) + np.uint64(1)
    cnt = rng.integers(0, 2**50, 50, dtype=np.uint64)
    limbs = rt.pack_limbs(cnt, hi, lo)
    c2, hi2, lo2 = rt.unpack_limbs(8 * limbs)
    assert np.array_equal(c2, 8 * cnt)
    for a, b, c, d in zip(hi, lo, hi2, lo2):
        assert (int(c) << 64 | int(d)) == 8 * (int(a) << 64 | int(b))
    # negative totals (two's complement, e.g. a bin whose terms are all 1 - ulp):
    # -5 on each of 3 ranks sums to -15 = (2^64 - 1) : (2^64 - 15)
    m1 = np.array([np.uint64(2**64 - 1)], dtype=np.uint64)
    neg = np.array([np.uint64(2**64 - 5)], dtype=np.uint64)
    limbs = rt.pack_limbs(np.zeros(1, np.uint64), m1, neg)
    _, hi3, lo3 = rt.unpack_limbs(3 * limbs)
    assert int(hi3[0]) == 2**64 - 1 and int(lo3[0]) == 2**64 - 15
    # mixed signs across ranks: +7, -2, -9 -> -4
    vals = [7, -2, -9]
    parts = [rt.pack_limbs(np.zeros(1, np.uint64),
                           np.array([np.uint64((v >> 64) & (2**64 - 1))], np.uint64),
                           np.array([np.uint64(v & (2**64 - 1))], np.uint64)) for v in vals]
    _, h4, l4 = rt.unpack_limbs(sum(parts))
    assert (int(h4[0]) << 64 | int(l4[0])) == (-4) % 2**128


def test_device_calls_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    region = geom.StudyRegion([[0, 0], [10, 0], [10, 10], [0, 10]], 0, 100)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        est.estimate_surface(([1.0, 2.0], [1.0, 2.0], [1, 2]), region, est.DistanceGrid([5.0], [5]))


def test_configs_generators_deterministic():
    from paper_1912_04753_b200 import configs

    c2 = configs.CONFIGS["C2"]
    a = configs.thomas(c2)
    b = configs.thomas(c2)
    assert all(np.array_equal(u, v) for u, v in zip(a, b))
    assert 90_000 < len(a[0]) < 110_000
    assert a[2].dtype == np.int64 and a[2].min() >= 0 and a[2].max() <= c2.period_s
    c4 = configs.CONFIGS["C4"]
    small = configs.Config("C4s", 20_000, c4.extent_m, c4.period_s, c4.s_step, c4.s_max,
                           c4.t_step, c4.t_max, 0, 4, "poi")
    x, y, t = configs.poi(small)
    assert len(x) == 20_000
    assert x.min() >= 0 and x.max() <= c4.extent_m and t.min() >= 0 and t.max() <= c4.period_s
    s, tv = configs.grid_values(configs.CONFIGS["C5"])
    assert len(s) == 50 and len(tv) == 50 and tv[-1] == 30 * 86400


def test_bench_reference_arm_contract():
    """`bench.py --impl reference` (the reference's own CPU path, oracle/_ref)
    prints one JSON line with the driver's contract keys (C1: seconds)."""
    import json
    import subprocess
    import sys

    import oracle

    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built here")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference",
                        "--config", "C1", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, timeout=600, cwd=root)
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads(p.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "reference"
    assert line["config"]["workload"].startswith("C1")
