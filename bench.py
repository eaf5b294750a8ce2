#!/usr/bin/env python
"""Benchmark of the space-time K pair path (BASELINE.json metric: space-time
pairs evaluated/s and K realisations/s vs roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C2]

A step is one whole rt::run_job of the workload (default configs[1] = C2: the
observed Thomas pattern + 99 CSR realisations, their K/L surfaces and the
envelopes).  ``value`` = in-threshold ordered pairs evaluated per second over
all ranks with the observed pattern already in HBM; ``e2e`` = the same through
the host-buffer C ABI call (``stk_run_job`` / ``stk_run_job_shard``: H2D of the
points and D2H of K, L, envelopes and diff inside the timed region).

Multi-GPU (torchrun, one process per GPU): the job is split strong-scaling
style — each rank takes a 1/N slice of the observed pattern's pair work and a
contiguous block of realisations; two exact all-reduces (SUM of integer
partials, MAX/MIN of envelopes) over NCCL combine them.

``--impl reference`` times the reference's own CPU implementation
(oracle/_ref: the unmodified reference sources, rt::run_job with a
LocalExecutor on all host threads) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# Algorithmic FP64 instruction budget per in-threshold pair (frozen):
W_INT = 22    # interior pair (omega == 1)
W_ARC = 600   # boundary-crossing pair (4-vertex polygon arc weight)
GRID_BYTES_PER_POINT = 88  # K1 algorithmic bytes per point


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--sims", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-sims", type=int, default=1)
    ap.add_argument("--cpu-sample-frac", type=float, default=1.0,
                    help="CPU reference sample: every (1/frac)-th observed point (pairs/s is "
                         "per pair, so a subsample keeps the metric comparable)")
    ap.add_argument("--n", type=int, default=0,
                    help="profiling only: replace the config's N (the line then names the "
                         "reduced N; not a headline measurement)")
    ap.add_argument("--ring", type=int, default=0,
                    help="replace the square by a regular polygon of this many vertices "
                         "(acceptance criterion 6 shape)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def workload(cfg_name, sims_override=None, ring_vertices=0, n_override=0):
    import dataclasses

    from paper_1912_04753_b200 import configs

    cfg = configs.CONFIGS[cfg_name]
    if n_override:
        cfg = dataclasses.replace(cfg, n=int(n_override))
    if ring_vertices:
        cfg = cfg.with_ring(ring_vertices)
    s, tv = configs.grid_values(cfg)
    sims = cfg.sims if sims_override is None else sims_override
    return cfg, s, tv, sims


def observed_points(cfg, dev=None):
    from paper_1912_04753_b200 import configs

    gen = None
    if cfg.kind == "csr":
        from paper_1912_04753_b200.stripley import geom, sim

        def gen(n, ring, p0, p1, seed):
            p = sim.generate_cstr(n, geom.StudyRegion(ring, p0, p1), seed, device=dev)
            return p.x, p.y, p.t
    return configs.observed(cfg, gen)


# ------------------------------------------------------------------ reference
def subsample(x, y, t, frac):
    k = max(1, int(round(1.0 / frac))) if frac < 1.0 else 1
    return x[::k], y[::k], t[::k]


def cpu_reference_step(x, y, t, cfg, s, tv, sample_sims, workers):
    """One bounded sample of the workload through the reference's rt::run_job."""
    from oracle import ref

    partitions = 4 * workers
    t0 = time.perf_counter()
    r = ref.run_job(x, y, t, cfg.ring(), 0, cfg.period_s, s, tv, sims=sample_sims, seed=cfg.seed,
                    method=0, partitions=partitions, workers=workers,
                    use_index=(cfg.name != "C3"), use_cache=False)
    dt = time.perf_counter() - t0
    return r["in_threshold"], dt


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cfg, s, tv, sims = workload(args.config, args.sims, args.ring, args.n)
    import oracle

    x, y, t = subsample(*observed_points_cpu(cfg), args.cpu_sample_frac)
    workers = os.cpu_count() or 1
    kind = "reference" if oracle.ref_available() else "port"
    if kind != "reference":
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref (reference compiled from source) not built"}))
        return
    sample_sims = args.cpu_sample_sims
    for _ in range(args.warmup):
        cpu_reference_step(x, y, t, cfg, s, tv, sample_sims, workers)
    pairs = 0
    secs = 0.0
    for _ in range(args.steps):
        p, dt = cpu_reference_step(x, y, t, cfg, s, tv, sample_sims, workers)
        pairs += p
        secs += dt
    value = pairs / secs
    sample = (f"{cfg.name} observed pattern ({len(x)} points) + {sample_sims} CSR realisation(s) per step "
              f"(of 1+{sims}), rt::run_job LocalExecutor({workers}), KDB {4 * workers} partitions, "
              f"index {'on' if cfg.name != 'C3' else 'off'}, cache off")
    line = {
        "impl": "reference", "metric": "space-time in-threshold pairs evaluated per second",
        "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_dict(cfg, sims, world),
        "realisations_per_s": args.steps * (1 + sample_sims) / secs,
        "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": workers, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def observed_points_cpu(cfg):
    from paper_1912_04753_b200 import configs

    gen = None
    if cfg.kind == "csr":
        from oracle import port

        gen = port.generate_cstr
    return configs.observed(cfg, gen)


def config_dict(cfg, sims, world):
    shape = (f"{cfg.ring_vertices}-vertex polygon inscribed in a {cfg.extent_m:g} m square"
             if cfg.ring_vertices else f"{cfg.extent_m:g} m square")
    return {"workload": f"{cfg.name}: {cfg.kind} N={cfg.n} in {shape} x "
                        f"{cfg.period_s} s, grid {cfg.s_max:g} m/{cfg.t_max} s, 1 observed + "
                        f"{sims} CSR realisations (rt::run_job)",
            "n_points": cfg.n, "realisations": 1 + sims, "parallelism": f"realisations+pairs x{world}",
            "l2": "inputs larger than L2 (each step generates and grids 1+sims patterns, "
                  "hundreds of MB)"}


# ------------------------------------------------------------------ ours
def run_ours(args):
    import torch

    from paper_1912_04753_b200 import _lib
    from paper_1912_04753_b200.stripley import device as devmod
    from paper_1912_04753_b200.stripley import est, geom, rt

    rank, world, local = dist_env()
    # STK_BENCH_DEVICE / STK_DIST_BACKEND let the multi-rank path be exercised
    # on one GPU with gloo (host-side reductions only, no cross-rank kernels)
    local = int(os.environ.get("STK_BENCH_DEVICE", local))
    backend = os.environ.get("STK_DIST_BACKEND", "nccl")
    torch.cuda.set_device(local)
    group = None
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        group = dist.group.WORLD
    dev = devmod.get(local)
    lib = dev.lib
    cfg, s, tv, sims = workload(args.config, args.sims, args.ring, args.n)
    region = geom.StudyRegion(cfg.ring(), 0, cfg.period_s)
    grid = est.DistanceGrid(s, tv)
    dev.configure(region, grid)
    x, y, t = observed_points(cfg, dev)
    n = len(x)
    shape = (len(s), len(tv))
    bins = shape[0] * shape[1]
    dx = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    dy = torch.from_numpy(np.ascontiguousarray(y)).cuda()
    dt = torch.from_numpy(np.ascontiguousarray(t)).cuda()
    hx = torch.from_numpy(np.ascontiguousarray(x)).pin_memory()
    hy = torch.from_numpy(np.ascontiguousarray(y)).pin_memory()
    ht = torch.from_numpy(np.ascontiguousarray(t)).pin_memory()
    stream = torch.cuda.ExternalStream(dev.stream_handle())
    executor = rt.DeviceExecutor(device=dev, rank=rank, world=world, group=group)
    r0, r1 = executor.sim_range(sims)
    spec = rt.JobSpec(grid=grid, sims=sims, seed=cfg.seed)

    out = {k: np.zeros(shape) for k in ("k", "l", "up", "lo", "diff")}
    cnt = np.zeros(shape, np.uint64)
    shi = np.zeros(shape, np.uint64)
    slo = np.zeros(shape, np.uint64)
    P = _lib.ptr

    def step(device_resident: bool):
        tel = _lib.StkTelemetry()
        if world == 1:
            if device_resident:
                rc = lib.stk_run_job_device(dev.h, dx.data_ptr(), dy.data_ptr(), dt.data_ptr(), n,
                                            sims, cfg.seed, 0, P(out["k"]), P(out["l"]),
                                            P(out["up"]), P(out["lo"]), P(out["diff"]),
                                            C.byref(tel))
            else:
                rc = lib.stk_run_job(dev.h, P(hx.numpy()), P(hy.numpy()),
                                     P(ht.numpy(), C.c_int64), n, sims, cfg.seed, 0, P(out["k"]),
                                     P(out["l"]), P(out["up"]), P(out["lo"]), P(out["diff"]),
                                     C.byref(tel))
            dev.check(rc)
        else:
            out["up"].fill(-np.inf)
            out["lo"].fill(np.inf)
            if device_resident:
                rc = lib.stk_run_job_shard_device(
                    dev.h, dx.data_ptr(), dy.data_ptr(), dt.data_ptr(), n, rank, world, r0, r1,
                    cfg.seed, 0, P(cnt, C.c_uint64), P(shi, C.c_uint64), P(slo, C.c_uint64),
                    P(out["up"]), P(out["lo"]), C.byref(tel))
            else:
                rc = lib.stk_run_job_shard(
                    dev.h, P(hx.numpy()), P(hy.numpy()), P(ht.numpy(), C.c_int64), n, rank, world,
                    r0, r1, cfg.seed, 0, P(cnt, C.c_uint64), P(shi, C.c_uint64),
                    P(slo, C.c_uint64), P(out["up"]), P(out["lo"]), C.byref(tel))
            dev.check(rc)
            rt._combine_ranks(executor, region, grid, n, spec, cnt, shi, slo, out["up"],
                              out["lo"], tel, time.perf_counter(), dev)
        return tel

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
        torch.cuda.synchronize()

    def timed(device_resident, steps):
        tels = []
        barrier()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(steps):
            tels.append(step(device_resident))
        ev1.record(stream)
        barrier()
        ms = ev0.elapsed_time(ev1)
        return ms, tels

    for _ in range(args.warmup):
        step(True)
    clocks = ClockSampler(local)
    clocks.start()
    ms, tels = timed(True, args.steps)
    clk = clocks.stop()
    step(False)  # the host-buffer path's own warm-up (its upload staging buffers)
    e2e_ms, e2e_tels = timed(False, args.steps)

    pairs_rank = sum(t_.in_threshold_pairs for t_ in tels)
    arc_rank = sum(t_.arc_pairs for t_ in tels)  # omega != 1 (SURVEY 8(d) arc pairs)
    exact_rank = sum(t_.exact_path_pairs for t_ in tels)
    cand_rank = sum(t_.candidate_pairs for t_ in tels)  # unordered pairs the kernel tested
    pair_ms_rank = sum(t_.pair_ms for t_ in tels)
    grid_ms_rank = sum(t_.grid_ms for t_ in tels)
    patterns_rank = sum(t_.patterns for t_ in tels)
    launches = sum(t_.kernel_launches for t_ in tels) // max(args.steps, 1)

    # max over ranks of time, sum over ranks of work
    tot = np.array([pairs_rank, arc_rank, patterns_rank, exact_rank, cand_rank], dtype=np.float64)
    tmax = np.array([ms, e2e_ms, pair_ms_rank, grid_ms_rank], dtype=np.float64)
    if world > 1:
        import torch.distributed as dist

        dev_ = "cuda" if backend == "nccl" else "cpu"
        a = torch.from_numpy(tot).to(dev_)
        b = torch.from_numpy(tmax).to(dev_)
        dist.all_reduce(a, op=dist.ReduceOp.SUM)
        dist.all_reduce(b, op=dist.ReduceOp.MAX)
        tot, tmax = a.cpu().numpy(), b.cpu().numpy()
    pairs, arcs, patterns, exact, cands = tot
    ms, e2e_ms, pair_ms, grid_ms = tmax

    if rank != 0:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()
        return

    value = pairs / (ms * 1e-3)
    e2e_value = pairs / (e2e_ms * 1e-3)
    peak = dev.fp64_peak()
    # roofline of the pair kernel: algorithmic FP64 instructions / pair-kernel time
    instr = (pairs - arcs) * W_INT + arcs * W_ARC
    achieved = instr / (pair_ms * 1e-3) if pair_ms > 0 else 0.0
    grid_gbs = (GRID_BYTES_PER_POINT * n * patterns) / (grid_ms * 1e-3) / 1e9 if grid_ms else None
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        hbm_peak = peaks.get("hbm_gbs")
    except Exception:
        hbm_peak = None

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, s, tv, sims, *subsample(x, y, t, args.cpu_sample_frac),
                           args.cpu_sample_sims)

    line = {
        "metric": "space-time in-threshold pairs evaluated per second",
        "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(cfg, sims, world),
        "realisations_per_s": patterns / (ms * 1e-3),
        "pairs_per_step": pairs / args.steps,
        "arc_fraction": arcs / pairs if pairs else None,
        "exact_path_fraction": exact / pairs if pairs else None,
        # secondary, implementation-dependent: (center, neighbour)
        # candidates the pair kernel tested, each serving both ordered pairs
        "candidate_pairs_per_s": cands / (ms * 1e-3),
        "candidates_per_unordered_in_threshold_pair": (2 * cands / pairs) if pairs else None,
        "e2e": {"value": e2e_value, "unit": "pairs/s",
                "h2d_bytes_per_step": int(24 * n),
                "d2h_bytes_per_step": int(8 * bins * (5 if world == 1 else 0) +
                                          (8 * bins * 5 if world > 1 else 0)),
                "realisations_per_s": patterns / (e2e_ms * 1e-3)},
        "roofline": {"bound": "fp64", "achieved": achieved / 1e12, "peak": peak / 1e12,
                     "unit": "FP64 Tinstr/s", "frac": achieved / peak if peak else None,
                     "traffic": ncu_capture(cfg.name)[0],
                     "hw": hw_view(ncu_capture(cfg.name)[1], pairs / args.steps, peak),
                     "note": f"pair kernel: ({W_INT} x interior + {W_ARC} x arc (omega != 1) pairs) "
                             "FP64 instr / CUDA-event pair-kernel time; peak = live DFMA "
                             "microbenchmark (stk_measure_fp64_peak)",
                     "kernel_ms_per_step": pair_ms / args.steps,
                     "grid_build": {"bound": "hbm", "achieved": grid_gbs, "peak": hbm_peak,
                                    "unit": "GB/s", "frac": (grid_gbs / hbm_peak)
                                    if grid_gbs and hbm_peak else None,
                                    "ms_per_step": grid_ms / args.steps}},
        "clocks": clk,
        "gpu_launches": int(launches * args.steps),
        "cpu_baseline": cpu,
    }
    print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def hw_view(hw, pairs_per_launch, peak):
    """SASS-counted FP64 instructions per in-threshold pair and the FP64 rate
    they imply over the captured launch (one pair-kernel launch per step)."""
    if hw and hw.get("fp64_thread_instructions") and pairs_per_launch:
        f = hw["fp64_thread_instructions"]
        hw["fp64_sass_instr_per_pair"] = f / pairs_per_launch
        hw["fp64_sass_rate_frac"] = (f / (hw["duration_ms"] * 1e-3)) / peak if peak else None
    return hw


def ncu_capture(cfg_name):
    """Per-launch figures of the pair kernel from the committed ncu capture of
    this workload (profiles/pair_kernel_ncu_r1.json, keyed by config): DRAM
    bytes read + written and the SM issue / FP64-pipe utilisation, or None."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "pair_kernel_ncu_r1.json")))[cfg_name]
    except Exception:
        return None, None
    hw = {"bound": "issue", "issue_active": d["issue_active"],
          "fp64_pipe_active": d["fp64_pipe_active"], "warps_active": d["warps_active"],
          "fp64_thread_instructions": d.get("fp64_thread_instructions"),
          "duration_ms": d["duration_ms"], "source": d["capture"]}
    return d["dram_bytes_read"] + d["dram_bytes_write"], hw


def cpu_baseline(cfg, s, tv, sims, x, y, t, sample_sims):
    try:
        import oracle

        if not oracle.ref_available():
            return {"value": None, "unit": "pairs/s", "cores": 0, "kind": "reference",
                    "sample": "oracle/_ref not built"}
        workers = os.cpu_count() or 1
        pairs, dt = cpu_reference_step(x, y, t, cfg, s, tv, sample_sims, workers)
        return {"value": pairs / dt, "unit": "pairs/s", "cores": workers, "kind": "reference",
                "sample": f"{cfg.name} observed ({len(x)} points) + {sample_sims} CSR realisation(s) through the "
                          f"reference rt::run_job, LocalExecutor({workers}), {dt:.1f} s"}
    except Exception as e:  # the baseline is reported, never the target
        return {"value": None, "unit": "pairs/s", "cores": 0, "kind": "reference",
                "sample": f"failed: {e}"}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
