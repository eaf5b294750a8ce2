"""Randomised differential test: the CUDA path against the oracle's C restatement on
small random jobs (regions, periods, grids, patterns).  Counts must be bit-exact,
weighted histograms and K within 1e-9 relative.
    python tests/fuzz_gpu.py [cases] [first_seed]
Prints one line per failure and a summary; exit code 1 on any failure."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


BIG = os.environ.get("FUZZ_BIG") == "1"  # larger patterns, polygons of up to 200 vertices


def random_case(seed):
    rng = np.random.default_rng(seed)
    kind = rng.choice(["rect", "rect", "rect", "poly"])
    off = float(rng.choice([0.0, 0.0, 1.0e3, -2.5e4, 5.0e5, 4.2e6]))
    w = float(10.0 ** rng.uniform(0.5, 4.5))
    h = w * float(rng.choice([1.0, 1.0, 0.37, 3.0, 0.05, 17.0]))
    if kind == "rect":
        ring = np.array([[off, off * 0.5], [off + w, off * 0.5], [off + w, off * 0.5 + h],
                         [off, off * 0.5 + h]])
    else:
        nv = int(rng.integers(3, 201 if BIG else 41))
        ang = np.sort(rng.uniform(0.0, 2.0 * np.pi, nv))
        while np.min(np.diff(np.concatenate([ang, [ang[0] + 2 * np.pi]]))) < 1e-3:
            ang = np.sort(rng.uniform(0.0, 2.0 * np.pi, nv))
        ring = np.stack([off + 0.5 * w * (1 + np.cos(ang)), off * 0.5 + 0.5 * h * (1 + np.sin(ang))],
                        axis=1)
    p0 = int(rng.choice([0, 0, -86400 * 1000, 1_600_000_000]))
    dur = int(rng.choice([59, 10_000, 31_536_000, 31_536_000, 2 ** 33 + 12345]))
    p1 = p0 + dur
    n = int(rng.choice([6000, 12000, 20000, 30000] if BIG else [2, 3, 17, 200, 1000, 2500, 4000, 12000]))
    extent = max(w, h)
    s_max = float(min(w, h) * 10.0 ** rng.uniform(-2.0, 0.3))
    cs = int(rng.integers(1, 26))
    if rng.random() < 0.75:
        s = s_max * np.arange(1, cs + 1) / cs
    else:
        s = np.sort(rng.uniform(0.02 * s_max, s_max, cs))
        s = np.unique(s)
    t_max = max(1, int(dur * 10.0 ** rng.uniform(-2.0, 0.1)))
    ct = int(rng.integers(1, 26))
    if rng.random() < 0.75:
        step = max(1, t_max // ct)
        tv = np.arange(1, ct + 1, dtype=np.int64) * step
    else:
        tv = np.unique(rng.integers(1, max(2, t_max), ct).astype(np.int64))
    cluster = float(rng.choice([1.0, 1.0, 0.3, 0.05]))
    return dict(ring=ring, p0=p0, p1=p1, n=n, s=np.ascontiguousarray(s, dtype=np.float64),
                tv=np.ascontiguousarray(tv, dtype=np.int64), cluster=cluster, kind=kind,
                pseed=int(rng.integers(1, 2 ** 62)), extent=extent,
                sims=int(rng.choice([0, 0, 0, 1, 4])), jseed=int(rng.integers(1, 2 ** 63)))


def points(case, port):
    x, y, t = port.generate_cstr(case["n"], case["ring"], case["p0"], case["p1"], case["pseed"])
    a = case["cluster"]
    if a < 1.0 and len(x) > 4:  # pull towards a few of the pattern's own points (convex regions)
        rng = np.random.default_rng(case["pseed"] & 0xffffffff)
        k = rng.integers(0, len(x), len(x) // 50 + 1)
        own = k[rng.integers(0, len(k), len(x))]
        x = x[own] + (x - x[own]) * a
        y = y[own] + (y - y[own]) * a
        t = (t[own] + np.rint((t - t[own]) * a)).astype(np.int64)
        t = np.clip(t, case["p0"], case["p1"])
        # rounding can push a pulled point across the boundary: keep valid inputs only
        keep = np.array([port.point_in_polygon(px, py, case["ring"]) for px, py in zip(x, y)])
        x, y, t = x[keep], y[keep], t[keep]
    return np.ascontiguousarray(x), np.ascontiguousarray(y), np.ascontiguousarray(t)


def run(cases, first, verbose=True):
    from conftest import rel_err, surfaces_close
    from oracle import port
    from paper_1912_04753_b200.stripley import est, geom, rt, sim

    bad = 0
    done = 0
    t0 = time.time()
    for seed in range(first, first + cases):
        c = random_case(seed)
        try:
            x, y, t = points(c, port)
            if len(x) < 2:
                continue
            region = geom.StudyRegion(c["ring"], c["p0"], c["p1"])
            grid = est.DistanceGrid(c["s"], c["tv"])
            o = port.estimate(x, y, t, c["ring"], c["p0"], c["p1"], c["s"], c["tv"])
            h = est.pair_histogram((x, y, t), region, grid)
            k = est.estimate_surface((x, y, t), region, grid)
        except Exception as e:  # both sides reject the same inputs, or a real error
            print(f"seed {seed}: {type(e).__name__}: {str(e)[:120]}")
            bad += 1
            continue
        done += 1
        ok_job = True
        if c["sims"] and c["n"] <= 4000:  # rt::run_job: realisations, envelopes, totals
            spec = rt.JobSpec(grid=grid, sims=c["sims"], seed=c["jseed"])
            small = c["sims"] >= 4 and (seed % 3 == 0)  # force several batches (budget ~2 patterns)
            from paper_1912_04753_b200.stripley import device as _device
            dev0 = _device.get(0)
            if small:
                dev0.set_memory_budget(max(1 << 20, 260 * len(x) + 64 * grid.cells_s() * grid.cells_t()))
            try:
                res = rt.run_job((x, y, t), region, spec, rt.DeviceExecutor(device=0))
            finally:
                if small:
                    dev0.set_memory_budget(16 << 30)
            ls, total = [], int(o["in_threshold"])
            for r in range(c["sims"]):
                sx, sy, st = port.generate_cstr(len(x), c["ring"], c["p0"], c["p1"],
                                                (c["jseed"] + r) % (2 ** 64))
                e = port.estimate(sx, sy, st, c["ring"], c["p0"], c["p1"], c["s"], c["tv"])
                ls.append(e["l"])
                total += int(e["in_threshold"])
            up, lo = port.envelopes(np.stack(ls))
            fl = np.isfinite(up) & np.isfinite(lo)
            tol = 1e-9 * max(1.0, float(np.max(np.abs(up[fl])))) if fl.any() else 0.0
            ok_job = (res.telemetry.in_threshold_pairs == total and
                      np.all(np.abs(np.where(fl, res.upper_l.values - up, 0.0)) <= tol) and
                      np.all(np.abs(np.where(fl, res.lower_l.values - lo, 0.0)) <= tol))
        rng = np.random.default_rng(seed)
        if rng.random() < 0.25:  # shards of the pattern's pair work sum exactly to the whole
            ns = int(rng.choice([2, 3, 5]))
            parts = [est.pair_histogram((x, y, t), region, grid, shard=k_, nshards=ns)
                     for k_ in range(ns)]
            tot_c = sum(p_["counts"].astype(object) for p_ in parts)
            tot_s = sum((p_["sum_hi"].astype(object) << 64) + p_["sum_lo"].astype(object)
                        for p_ in parts) % (1 << 128)
            whole = (h["sum_hi"].astype(object) << 64) + h["sum_lo"].astype(object)
            # a bin that received 1/0 carries + 2^120 per partial holding such a pair
            # (stk.h: any sum >= 2^119 finalizes to NaN): compare mark and value apart
            mark = lambda v: np.array([int(a) >= (1 << 119) for a in v.ravel()])
            low = lambda v: np.array([int(a) % (1 << 119) for a in v.ravel()], dtype=object)
            ok_job = ok_job and bool(np.all(tot_c == h["counts"].astype(object))) and \
                bool(np.all(mark(tot_s) == mark(whole))) and bool(np.all(low(tot_s) == low(whole)))
        if rng.random() < 0.25 and c["n"] <= 4000:  # bootstrap / permutation null models
            method = sim.Method.Bootstrap if rng.random() < 0.5 else sim.Method.Permutation
            gen = port.generate_bootstrap if method == sim.Method.Bootstrap else \
                port.generate_permutation
            l_all, _, _ = sim.simulate((x, y, t), region, grid, method, 0, 2, c["jseed"])
            for r in range(2):
                bx, by, bt = gen(x, y, t, (c["jseed"] + r) % (2 ** 64))
                e = port.estimate(bx, by, bt, c["ring"], c["p0"], c["p1"], c["s"], c["tv"])
                fl = np.isfinite(e["l"])
                tol = 1e-9 * max(1.0, float(np.max(np.abs(e["l"][fl])))) if fl.any() else 0.0
                ok_job = ok_job and bool(np.all(np.abs(np.where(fl, l_all[r] - e["l"], 0.0)) <= tol))
        ok_counts = np.array_equal(h["counts"], o["counts"])
        fin = np.isfinite(o["k"])
        ok_k = surfaces_close(np.where(fin, k.values, 0.0), np.where(fin, o["k"], 0.0), 1e-9) and \
            np.array_equal(np.isfinite(k.values), fin)
        if not (ok_counts and ok_k and ok_job):
            bad += 1
            print(f"seed {seed}: job {'ok' if ok_job else 'DIFFERS'} counts {'ok' if ok_counts else 'DIFFER'} K "
                  f"{'ok' if ok_k else 'DIFFERS'} kind={c['kind']} n={c['n']} cs={len(c['s'])} "
                  f"ct={len(c['tv'])} dur={c['p1'] - c['p0']} cluster={c['cluster']}")
    if verbose:
        print(f"fuzz: {done} cases compared, {bad} failures, {time.time() - t0:.1f} s")
    return done, bad


if __name__ == "__main__":
    _, nbad = run(int(sys.argv[1]) if len(sys.argv) > 1 else 100,
                  int(sys.argv[2]) if len(sys.argv) > 2 else 1)
    sys.exit(1 if nbad else 0)
