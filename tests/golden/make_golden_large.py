"""Full-size parity fixtures for the BASELINE configs, produced by the reference.

Run HERE (the container with /root/reference; hours of CPU for C3/C5):

    nice -n 19 python tests/golden/make_golden_large.py [C2 C4 C3 C5] [--workers 8]

Each config writes one small .npz under tests/golden/ as soon as it finishes:

* ``c2_job.npz``  -- the whole C2 job (observed Thomas pattern + 99 CSR
  realisations) through the reference's ``rt::run_job`` + ``LocalExecutor``
  (proj/core/src/runtime.cpp:190-249): K, L, upper, lower, diff and the job's
  in-threshold total; per-bin counts of the observed pattern.
* ``c3_full.npz`` -- C3 at full N = 200,000 (single realisation): K, L,
  in-threshold total, per-bin counts.
* ``c4_parity.npz`` / ``c5_parity.npz`` -- the observed pattern plus
  realisations r in {0, 1, m/2, m-1} at full N (SURVEY §8(c)'s budget):
  per pattern K, L, in-threshold total and per-bin counts, plus the envelope
  over that subset.  Each pattern goes through ``rt::run_job``'s own loop body
  (``oracle.ref.Job``: plan once on the observed points, then
  make_tasks -> executor.run -> aggregate -> to_l; realisation r is
  ``sim::generate(Cstr, n, ..., seed + r)``).

Per-bin counts come from the reference's own STR R-tree query plus
``geom::spatial_distance`` / ``temporal_distance`` / ``est::bin_pair``
(``oracle.ref.pair_counts_indexed``); their total is checked against the
reference's ``in_threshold_pairs``.  Observed patterns are regenerated on the
GPU box by ``configs.observed`` (seeded numpy for C2/C4/C5, the device CSR
generator for C3), so each fixture stores the pattern's n and coordinate sums
to prove the regenerated input is the same.
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from oracle import ref  # noqa: E402
from paper_1912_04753_b200 import configs  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def log(msg):
    print(time.strftime("%H:%M:%S"), msg, flush=True)


def fingerprint(x, y, t):
    return dict(n=len(x), sum_x=float(np.sum(x)), sum_y=float(np.sum(y)),
                sum_t=int(np.sum(t.astype(np.int64))))


def setup(name):
    cfg = configs.CONFIGS[name]
    s, tv = configs.grid_values(cfg)
    ring = cfg.ring()
    x, y, t = configs.observed(cfg, csr_generator=ref.generate_cstr)
    return cfg, s, tv, ring, x, y, t


def c2_job(workers):
    cfg, s, tv, ring, x, y, t = setup("C2")
    log(f"C2: n={len(x)} full job 1+{cfg.sims}")
    t0 = time.time()
    r = ref.run_job(x, y, t, ring, 0, cfg.period_s, s, tv, sims=cfg.sims, seed=cfg.seed,
                    partitions=4 * workers, workers=workers, use_index=True, use_cache=False)
    log(f"C2 job {time.time() - t0:.0f}s in_threshold={r['in_threshold']}")
    counts = ref.pair_counts_indexed(x, y, t, s, tv, threads=workers)
    job = ref.Job(x, y, t, ring, 0, cfg.period_s, s, tv, seed=cfg.seed,
                  partitions=4 * workers, workers=workers)
    obs = job.pattern(-1)
    job.close()
    assert int(counts.sum()) == obs["in_threshold"], (counts.sum(), obs["in_threshold"])
    np.savez_compressed(os.path.join(OUT, "c2_job.npz"), k=r["k"], l=r["l"], upper=r["upper"],
                        lower=r["lower"], diff=r["diff"], in_threshold_total=r["in_threshold"],
                        counts_observed=counts, in_threshold_observed=obs["in_threshold"],
                        s=s, tv=tv, seed=cfg.seed, sims=cfg.sims, **fingerprint(x, y, t))
    log("C2 written")


def c3_full(workers):
    cfg, s, tv, ring, x, y, t = setup("C3")
    log(f"C3: n={len(x)} single realisation, all pairs")
    t0 = time.time()
    counts = ref.pair_counts_indexed(x, y, t, s, tv, threads=workers)
    log(f"C3 counts {time.time() - t0:.0f}s total={int(counts.sum())}")
    t0 = time.time()
    r = ref.run_job(x, y, t, ring, 0, cfg.period_s, s, tv, sims=0, seed=cfg.seed,
                    partitions=4 * workers, workers=workers, use_index=True, use_cache=False)
    log(f"C3 job {time.time() - t0:.0f}s in_threshold={r['in_threshold']}")
    assert int(counts.sum()) == r["in_threshold"]
    np.savez_compressed(os.path.join(OUT, "c3_full.npz"), k=r["k"], l=r["l"],
                        in_threshold=r["in_threshold"], counts=counts, s=s, tv=tv,
                        **fingerprint(x, y, t))
    log("C3 written")


def subset_parity(name, workers):
    cfg, s, tv, ring, x, y, t = setup(name)
    m = cfg.sims
    rs = [0, 1, m // 2, m - 1]
    log(f"{name}: n={len(x)} observed + realisations {rs}")
    job = ref.Job(x, y, t, ring, 0, cfg.period_s, s, tv, seed=cfg.seed,
                  partitions=4 * workers, workers=workers)
    out = dict(s=s, tv=tv, seed=cfg.seed, sims=m, realisations=np.array(rs),
               **fingerprint(x, y, t))
    path = os.path.join(OUT, f"{name.lower()}_parity.npz")
    if os.path.exists(path):  # resume: keep the patterns a previous run finished
        old = np.load(path)
        if all(np.array_equal(old[k], np.asarray(v)) for k, v in out.items()):
            out.update({k: old[k] for k in old.files})
    for which in [-1] + rs:
        key = "obs" if which < 0 else f"r{which}"
        if f"{key}_k" in out:
            log(f"{name} {key}: already in {os.path.basename(path)}")
            continue
        t0 = time.time()
        res = job.pattern(which)
        dt = time.time() - t0
        if which < 0:
            px, py, pt = x, y, t
        else:
            px, py, pt = ref.generate_cstr(len(x), ring, 0, cfg.period_s, cfg.seed + which)
        t1 = time.time()
        counts = ref.pair_counts_indexed(px, py, pt, s, tv, threads=workers)
        log(f"{name} {key}: job {dt:.0f}s counts {time.time() - t1:.0f}s "
            f"in_threshold={res['in_threshold']}")
        assert int(counts.sum()) == res["in_threshold"], (counts.sum(), res["in_threshold"])
        out[f"{key}_k"] = res["k"]
        out[f"{key}_l"] = res["l"]
        out[f"{key}_in_threshold"] = res["in_threshold"]
        out[f"{key}_counts"] = counts
        out[f"{key}_seconds"] = dt
        np.savez_compressed(path, **out)  # checkpoint after every pattern
    job.close()
    ls = np.stack([out[f"r{r}_l"] for r in rs])
    out["upper_subset"] = ls.max(0)
    out["lower_subset"] = ls.min(0)
    np.savez_compressed(path, **out)
    log(f"{name} written")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["C2", "C4", "C3", "C5"])
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 8)
    a = ap.parse_args()
    oracle.build(with_ref=True)
    for c in a.configs:
        if c == "C2":
            c2_job(a.workers)
        elif c == "C3":
            c3_full(a.workers)
        else:
            subset_parity(c, a.workers)
