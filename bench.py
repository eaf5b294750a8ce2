#!/usr/bin/env python
"""Benchmark of the space-time K pair path (BASELINE.json metric: space-time
pairs evaluated/s and K realisations/s vs roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C2]

A step is one whole rt::run_job of the workload (default C4, the largest
BASELINE config whose full job fits one GPU and whose reference arm can be
timed per realisation at full N: the observed 1M-point POI pattern + 99 CSR
realisations, their K/L surfaces and the envelopes).  ``value`` = in-threshold ordered pairs evaluated per second over
all ranks with the observed pattern already in HBM; ``e2e`` = the same through
the host-buffer C ABI call (``stk_run_job`` / ``stk_run_job_shard``: H2D of the
points and D2H of K, L, envelopes and diff inside the timed region).

Multi-GPU (torchrun, one process per GPU): the job is split strong-scaling
style — each rank takes a 1/N slice of the observed pattern's pair work and a
contiguous block of realisations; one collective library call per step
(stk_run_job_dist) combines them with two exact NCCL all-reduces on device
buffers (SUM of integer limbs, MAX/MIN of envelopes) over the communicator the
library holds.

``--impl reference`` times the reference's own CPU implementation
(oracle/_ref: the unmodified reference sources, rt::run_job's own loop body
with a LocalExecutor on all host threads).  Each step is one pattern of the
same job at full N (the first timed step the observed pattern, then CSR
realisations r = 0, 1, ...); the line reports the full job extrapolated from
them: T_plan + T_obs + m * mean(T_csr).
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
# FP64 thread-instruction peak: 148 SMs x 64 FP64 lanes x f_clk
FP64_PEAK_AT_MAX = 148 * 64 * 1.965e9
F_MAX_HZ = 1.965e9
ISSUE_PER_CLK = 148 * 4  # warp-instructions issued per clock (4 schedulers per SM)
GRID_BYTES_PER_POINT = 88  # K1 algorithmic bytes per point


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--sims", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-sims", type=int, default=1,
                    help="CSR realisations in our line's cpu_baseline sample")
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


def ref_job(x, y, t, cfg, s, tv, workers):
    """The reference's rt::run_job planned once on the observed points (timed:
    build_plan is part of the job, runtime.cpp:200-204)."""
    from oracle import ref

    t0 = time.perf_counter()
    job = ref.Job(x, y, t, cfg.ring(), 0, cfg.period_s, s, tv, seed=cfg.seed, method=0,
                  partitions=4 * workers, workers=workers, use_index=(cfg.name != "C3"),
                  use_cache=False)
    return job, time.perf_counter() - t0


def ref_pattern(job, which):
    """One pattern of the job through rt::run_job's loop body (runtime.cpp:216-239):
    the observed pattern (which < 0) or CSR realisation `which` (seed + which),
    generation included.  Returns (in-threshold pairs, seconds)."""
    t0 = time.perf_counter()
    r = job.pattern(which)
    return r["in_threshold"], time.perf_counter() - t0


def extrapolate(t_plan, obs, csr, sims):
    """Full-job estimate from measured patterns: T = T_plan + T_obs + m * mean(T_csr),
    pairs = P_obs + m * mean(P_csr).  obs, csr: (pairs, seconds)."""
    p_obs, t_obs = obs
    if csr:
        p_csr = sum(p for p, _ in csr) / len(csr)
        t_csr = sum(d for _, d in csr) / len(csr)
    else:  # no realisation measured: the observed pattern's rate stands for them
        p_csr, t_csr = p_obs, t_obs
    secs = t_plan + t_obs + sims * t_csr
    return p_obs + sims * p_csr, secs


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cfg, s, tv, sims = workload(args.config, args.sims, args.ring, args.n)
    import oracle

    x, y, t = subsample(*observed_points_cpu(cfg), args.cpu_sample_frac)
    workers = os.cpu_count() or 1
    if not oracle.ref_available():
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref (reference compiled from source) not built"}))
        return
    # Wall budget of the whole arm (a C4 realisation takes ~8 s on 16 cores): the
    # warm-up stops after a fifth of it, the timed realisations when it is spent
    # (at least two are measured); the line says how many were.
    budget = float(os.environ.get("STK_REF_BUDGET_S", "240"))
    t_start = time.perf_counter()
    job, t_plan = ref_job(x, y, t, cfg, s, tv, workers)
    # warm-up: realisations from the top of the seed ladder (not reused below)
    for i in range(args.warmup):
        if i > 0 and time.perf_counter() - t_start > 0.2 * budget:
            break
        ref_pattern(job, max(sims - 1 - i, 0))
    obs = ref_pattern(job, -1)
    csr = []
    for r in range(max(args.steps - 1, 0)):
        if len(csr) >= 2 and time.perf_counter() - t_start > budget:
            break
        csr.append(ref_pattern(job, r))
    job.close()
    pairs, secs = extrapolate(t_plan, obs, csr, sims)
    value = pairs / secs
    measured = obs[1] + sum(d for _, d in csr)
    sample = (f"{cfg.name} at full N: observed pattern ({len(x)} points, {obs[1]:.2f} s) + "
              f"{len(csr)} CSR realisations (mean {extrapolate(0, obs, csr, 1)[1] - obs[1]:.2f} s) "
              f"through rt::run_job's loop body, plan {t_plan:.2f} s; full job of 1+{sims} "
              f"extrapolated as T_plan + T_obs + {sims} x mean(T_csr) = {secs:.1f} s; "
              f"LocalExecutor({workers}), KDB {4 * workers} partitions, "
              f"index {'on' if cfg.name != 'C3' else 'off'}, cache off")
    line = {
        "impl": "reference", "metric": "space-time in-threshold pairs evaluated per second",
        "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * measured / (1 + len(csr)),
        "steps_measured": 1 + len(csr),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_dict(cfg, sims, world),
        "realisations_per_s": (1 + sims) / secs,
        "job_seconds_extrapolated": secs,
        "pairs_per_job": pairs,
        "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": workers,
                         "kind": "reference", "sample": sample},
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
    # N > 1 over NCCL: the executor joins a communicator inside the library (the
    # unique id travels once over the torch.distributed group, outside timing)
    try:
        executor = rt.DeviceExecutor(device=dev, rank=rank, world=world, group=group,
                                     comm=(world > 1 and backend == "nccl"))
    except Exception as e:  # NCCL inside the library unavailable: host-group exchange
        print(f"bench: library communicator unavailable ({e}); exchanging over the "
              "torch.distributed group", file=sys.stderr)
        executor = rt.DeviceExecutor(device=dev, rank=rank, world=world, group=group, comm=False)
    r0, r1 = executor.sim_range(sims)
    spec = rt.JobSpec(grid=grid, sims=sims, seed=cfg.seed)

    out = {k: np.zeros(shape) for k in ("k", "l", "up", "lo", "diff")}
    cnt = np.zeros(shape, np.uint64)
    shi = np.zeros(shape, np.uint64)
    slo = np.zeros(shape, np.uint64)
    P = _lib.ptr

    def step(device_resident: bool):
        tel = _lib.StkTelemetry()
        if world == 1 or executor.comm:
            # one library call; at N > 1 a collective over the NCCL communicator
            # inside the library (stk_run_job_dist: this rank's shard of the
            # observed pattern + its block of realisations, exact device
            # all-reduces, device finalize)
            dist_ = executor.comm
            if device_resident:
                fn = lib.stk_run_job_dist_device if dist_ else lib.stk_run_job_device
                rc = fn(dev.h, dx.data_ptr(), dy.data_ptr(), dt.data_ptr(), n, sims, cfg.seed, 0,
                        P(out["k"]), P(out["l"]), P(out["up"]), P(out["lo"]), P(out["diff"]),
                        C.byref(tel))
            else:
                fn = lib.stk_run_job_dist if dist_ else lib.stk_run_job
                rc = fn(dev.h, P(hx.numpy()), P(hy.numpy()), P(ht.numpy(), C.c_int64), n, sims,
                        cfg.seed, 0, P(out["k"]), P(out["l"]), P(out["up"]), P(out["lo"]),
                        P(out["diff"]), C.byref(tel))
            dev.check(rc)
        else:
            # host-group emulation (STK_DIST_BACKEND=gloo: several ranks on one GPU)
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
    dev_ms_rank = sum(t_.total_ms for t_ in tels)  # device time inside the calls
    patterns_rank = sum(t_.patterns for t_ in tels)
    launches = sum(t_.kernel_launches for t_ in tels) // max(args.steps, 1)

    # max over ranks of time, sum over ranks of work
    tot = np.array([pairs_rank, arc_rank, patterns_rank, exact_rank, cand_rank], dtype=np.float64)
    tmax = np.array([ms, e2e_ms, pair_ms_rank, grid_ms_rank, dev_ms_rank], dtype=np.float64)
    if world > 1:
        import torch.distributed as dist

        dev_ = "cuda" if backend == "nccl" else "cpu"
        a = torch.from_numpy(tot).to(dev_)
        b = torch.from_numpy(tmax).to(dev_)
        dist.all_reduce(a, op=dist.ReduceOp.SUM)
        dist.all_reduce(b, op=dist.ReduceOp.MAX)
        tot, tmax = a.cpu().numpy(), b.cpu().numpy()
    pairs, arcs, patterns, exact, cands = tot
    ms, e2e_ms, pair_ms, grid_ms, dev_ms = tmax

    if rank != 0:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()
        return

    value = pairs / (ms * 1e-3)
    e2e_value = pairs / (e2e_ms * 1e-3)
    # SURVEY §8(d) roofline denominator at the clock observed during the timed
    # region: 148 SMs x 64 FP64 lanes x f_clk (1.86e13 /s at 1965 MHz)
    f_clk = (clk.get("sm_mhz") or clk.get("sm_max_mhz") or 1965.0) * 1e6
    peak = FP64_PEAK_AT_MAX * f_clk / F_MAX_HZ
    dfma = dev.fp64_peak()  # live DFMA micro-benchmark (side note)
    # roofline of the pair kernel: algorithmic FP64 instructions / pair-kernel time
    instr = (pairs - arcs) * W_INT + arcs * W_ARC
    achieved = instr / (pair_ms * 1e-3) if pair_ms > 0 else 0.0
    grid_gbs = (GRID_BYTES_PER_POINT * n * patterns) / (grid_ms * 1e-3) / 1e9 if grid_ms else None
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        hbm_peak = peaks.get("hbm_gbs")
    except Exception:
        hbm_peak = None
    cap = ncu_capture(cfg.name, n, sims)
    pair_rate = pairs / (pair_ms * 1e-3) if pair_ms > 0 else 0.0
    issue = None
    if cap and cap.get("warp_instructions") and pairs:
        wipp = cap["warp_instructions"] / (pairs / args.steps)  # per in-threshold ordered pair
        issue = {"bound": "issue", "warp_instr_per_pair": wipp,
                 "achieved": wipp * pair_rate / 1e12, "peak": ISSUE_PER_CLK * f_clk / 1e12,
                 "unit": "T warp-instr/s",
                 "frac": wipp * pair_rate / (ISSUE_PER_CLK * f_clk),
                 "note": "ncu warp-instructions per launch / in-threshold ordered pairs per "
                         "launch x the live pair rate / (148 SMs x 4 schedulers x f_clk)"}

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
        # device time between the call's first and last event (the rest of
        # ms_per_step is host-side: the ctypes call, launch / graph submission)
        "device_ms_per_step": dev_ms / args.steps,
        "pairs_per_step": pairs / args.steps,
        "arc_fraction": arcs / pairs if pairs else None,
        "exact_path_fraction": exact / pairs if pairs else None,
        # secondary, implementation-dependent: (center, neighbour)
        # candidates the pair kernel tested, each serving both ordered pairs
        "candidate_pairs_per_s": cands / (ms * 1e-3),
        "candidates_per_unordered_in_threshold_pair": (2 * cands / pairs) if pairs else None,
        "e2e": {"value": e2e_value, "unit": "pairs/s",
                "h2d_bytes_per_step": int(24 * n),
                "d2h_bytes_per_step": int(8 * bins * 5),  # K, L, upper, lower, diff
                "realisations_per_s": patterns / (e2e_ms * 1e-3)},
        "roofline": {"bound": "fp64", "achieved": achieved / 1e12, "peak": peak / 1e12,
                     "unit": "FP64 Tinstr/s", "frac": achieved / peak if peak else None,
                     "traffic": cap["dram_bytes"] if cap else None,
                     "note": f"pair kernel: ({W_INT} x interior + {W_ARC} x arc (omega != 1) "
                             "in-threshold pairs) FP64 instr / CUDA-event pair-kernel time; "
                             "peak = 148 SMs x 64 lanes x f_clk (SURVEY 8(d)) at the median "
                             "SM clock of the timed region; traffic = ncu DRAM bytes per launch "
                             "of the capture stamped with this build's source hash",
                     "f_clk_mhz": f_clk / 1e6, "dfma_microbench_peak": dfma / 1e12,
                     "kernel_ms_per_step": pair_ms / args.steps,
                     "issue": issue,
                     "hw": cap,
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


def ncu_capture(cfg_name, n, sims):
    """Per-launch hardware figures of the pair kernel from the committed ncu
    capture of this workload (profiles/pair_kernel_ncu.json, written by
    profiles/ncu_json.py): used only when the capture's source hash equals this
    build's (paper_1912_04753_b200.build.source_hash) and its workload matches;
    otherwise None (a stale capture is never reported)."""
    try:
        from paper_1912_04753_b200 import build

        d = json.load(open(os.path.join(ROOT, "profiles", "pair_kernel_ncu.json")))[cfg_name]
        if d.get("src_hash") != build.source_hash():
            return None
        if d.get("n") not in (None, n) or d.get("sims") not in (None, sims):
            return None
    except Exception:
        return None
    keys = ("issue_active", "fp64_pipe_active", "warps_active", "warp_instructions",
            "fp64_thread_instructions", "duration_ms", "capture", "src_hash")
    out = {k: d.get(k) for k in keys}
    out["dram_bytes"] = d["dram_bytes_read"] + d["dram_bytes_write"]
    return out


def cpu_baseline(cfg, s, tv, sims, x, y, t, sample_sims):
    """Our line's CPU baseline: the reference's rt::run_job loop body on all host
    cores, observed pattern + `sample_sims` CSR realisations at full N, the full
    job extrapolated as in the reference arm."""
    try:
        import oracle

        if not oracle.ref_available():
            return {"value": None, "unit": "pairs/s", "cores": 0, "kind": "reference",
                    "sample": "oracle/_ref not built"}
        workers = os.cpu_count() or 1
        job, t_plan = ref_job(x, y, t, cfg, s, tv, workers)
        obs = ref_pattern(job, -1)
        csr = [ref_pattern(job, r) for r in range(sample_sims)]
        job.close()
        pairs, secs = extrapolate(t_plan, obs, csr, sims)
        return {"value": pairs / secs, "unit": "pairs/s", "cores": workers, "kind": "reference",
                "realisations_per_s": (1 + sims) / secs,
                "sample": f"{cfg.name} observed ({len(x)} points, {obs[1]:.1f} s) + "
                          f"{len(csr)} CSR realisation(s) through the reference's rt::run_job "
                          f"loop body, LocalExecutor({workers}); full job of 1+{sims} "
                          f"extrapolated: {secs:.1f} s"}
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
