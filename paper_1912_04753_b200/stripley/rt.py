"""``stripley::rt`` mirror (proj/core/include/stripley/runtime.hpp).

``run_job`` keeps the reference's signature and result.  The reference plans
KDB partitions and ships tasks to an ``Executor`` (runtime.hpp:108-117); on the
device that decomposition is replaced by the on-device grid, so the executor
here is a ``DeviceExecutor``: one process per GPU, and, across processes,
``torch.distributed`` for the two real exchange steps of the path:

* the observed pattern's pair work is split into ``world`` disjoint slices
  (``stk_pair_histogram`` shards); exact integer partials are summed with one
  all-reduce (bit-identical at any GPU count);
* realisations ``[0, sims)`` are split into contiguous ranges; each rank
  produces its partial envelopes, combined with all-reduce MAX / MIN (exact).
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np

from .. import _lib
from . import device as _device
from .est import (DistanceGrid, EstimatorOptions, KSurface, SurfaceKind, _prepare,
                  finalize_exact, theoretical_surface)
from .geom import Points, StudyRegion, TimeUnit
from .sim import Method


class PartitionerChoice(IntEnum):  # runtime.hpp:18
    Kdb = 0
    Hash = 1


class Mode(IntEnum):  # runtime.hpp:19
    Local = 0
    Distributed = 1


@dataclass
class JobSpec:  # runtime.hpp:21-33
    grid: DistanceGrid = None
    method: Method = Method.Cstr
    sims: int = 99
    seed: int = 1
    options: EstimatorOptions = field(default_factory=EstimatorOptions)
    partitioner: PartitionerChoice = PartitionerChoice.Kdb
    partitions: int = 1
    workers: int = 1
    mode: Mode = Mode.Local
    sample_fraction: float = 0.01
    time_unit: TimeUnit = TimeUnit.Days


@dataclass
class RunTelemetry:  # runtime.hpp:59-72 (pair counters + timings)
    pair_comparisons: int = 0
    in_threshold_pairs: int = 0
    exact_path_pairs: int = 0
    plan_seconds: float = 0.0
    estimation_seconds: float = 0.0
    simulation_seconds: float = 0.0
    device_ms: float = 0.0
    pair_ms: float = 0.0


@dataclass
class RunResult:  # runtime.hpp:138-146
    k_hat: KSurface
    l_hat: KSurface
    theoretical: KSurface
    upper_l: KSurface | None = None
    lower_l: KSurface | None = None
    diff_upper: KSurface | None = None
    telemetry: RunTelemetry = field(default_factory=RunTelemetry)


class DeviceExecutor:
    """Executor backed by one GPU per process.

    ``rank``/``world`` default to torch.distributed's when it is initialised.
    With world > 1 on an NCCL process group (or ``comm=True``) the executor
    joins an NCCL communicator INSIDE the library (``stk_comm_init``; the
    unique id travels once over ``group``), and ``run_job`` is one collective
    library call (``stk_run_job_dist``: exact device all-reduces, finalize on
    the device).  Otherwise (a gloo group: CPU tests of the sharding logic, or
    several ranks emulated on one GPU) the two exact exchanges run over
    ``group`` from the host (:func:`allreduce_exact`, :func:`allreduce_envelopes`).
    """

    def __init__(self, device=None, rank=None, world=None, group=None, comm=None):
        self.device = device
        self.group = group
        if rank is None or world is None:
            rank, world = 0, 1
            try:
                import torch.distributed as dist

                if dist.is_available() and dist.is_initialized():
                    rank, world = dist.get_rank(group), dist.get_world_size(group)
            except Exception:
                pass
        self.rank, self.world = int(rank), int(world)
        if not (0 <= self.rank < self.world):
            raise ValueError("rank must be < world")
        self.comm = False
        if comm is None:
            comm = self.world > 1 and _group_backend(group) == "nccl"
        if comm:
            self._init_comm()

    def _dev(self):
        return self.device if isinstance(self.device, _device.Device) else _device.get(self.device)

    @property
    def device_index(self) -> int:
        return self._dev().index

    def _init_comm(self):
        d = self._dev()
        if self.world == 1:
            uid = _device.nccl_unique_id()
        else:
            import torch.distributed as dist

            box = [_device.nccl_unique_id() if self.rank == 0 else None]
            dist.broadcast_object_list(box, src=0, group=self.group)
            uid = box[0]
        d.comm_init(uid, self.world, self.rank)
        self.comm = True

    # ----------------------------------------------------------- sharding
    def sim_range(self, sims: int) -> tuple[int, int]:
        """Contiguous block of realisations owned by this rank."""
        return shard_range(sims, self.rank, self.world)

    def allreduce_exact(self, counts, hi, lo):
        return allreduce_exact(counts, hi, lo, self.group, self._torch_device())

    def allreduce_envelopes(self, upper, lower):
        return allreduce_envelopes(upper, lower, self.group, self._torch_device())

    def _torch_device(self):
        import torch

        if _group_backend(self.group) == "nccl":
            return torch.device("cuda", self.device_index)
        return torch.device("cpu")


def _group_backend(group):
    try:
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            return dist.get_backend(group)
    except Exception:
        pass
    return None


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    base, extra = divmod(total, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


_M32 = np.uint64(0xFFFFFFFF)


def pack_limbs(counts, hi, lo):
    """Exact per-bin partials -> int64 limbs whose plain integer SUM across
    ranks is exact: [counts, lo & (2^32-1), lo >> 32, hi] (32-bit halves cannot
    overflow below 2^31 ranks; hi is the signed high word of the two's
    complement 128-bit sum).  The same algebra as the device's
    pack_exact_kernel / unpack_exact_kernel (stk_kernels.cu)."""
    lo = np.asarray(lo, np.uint64)
    return np.stack([np.asarray(counts, np.uint64), lo & _M32, lo >> np.uint64(32),
                     np.asarray(hi, np.uint64)]).view(np.int64)


def unpack_limbs(limbs):
    """Inverse of :func:`pack_limbs` after the SUM (vectorised, wrapping
    uint64 arithmetic = arithmetic mod 2^128)."""
    u = np.asarray(limbs, np.int64).view(np.uint64)
    counts, l32, h32, hi = u[0], u[1], u[2], u[3]
    with np.errstate(over="ignore"):
        a = h32 << np.uint64(32)
        lo = a + l32
        hi = hi + (h32 >> np.uint64(32)) + (lo < a).astype(np.uint64)
    return counts, hi, lo


def allreduce_exact(counts, hi, lo, group=None, device=None):
    """Sum exact per-bin partials across ranks: counts (u64) and the 128-bit
    fixed-point sums as integer limbs, so the SUM carries every bit
    (bit-identical at any world size)."""
    import torch
    import torch.distributed as dist

    ten = torch.from_numpy(pack_limbs(counts, hi, lo)).to(device or "cpu")
    dist.all_reduce(ten, op=dist.ReduceOp.SUM, group=group)
    return unpack_limbs(ten.cpu().numpy())


def allreduce_envelopes(upper, lower, group=None, device=None):
    """Pointwise MAX of upper / MIN of lower across ranks (exact, order-free)."""
    import torch
    import torch.distributed as dist

    u = torch.from_numpy(np.ascontiguousarray(upper)).to(device or "cpu")
    l = torch.from_numpy(np.ascontiguousarray(lower)).to(device or "cpu")
    dist.all_reduce(u, op=dist.ReduceOp.MAX, group=group)
    dist.all_reduce(l, op=dist.ReduceOp.MIN, group=group)
    return u.cpu().numpy(), l.cpu().numpy()


def run_job(points, region: StudyRegion, spec: JobSpec, executor: DeviceExecutor | None = None
            ) -> RunResult:
    """``rt::run_job`` (runtime.cpp:190-249): estimate, simulate, envelope."""
    executor = executor or DeviceExecutor()
    grid = spec.grid
    pts, d = _prepare(points, region, grid, spec.options, executor.device)
    n = len(pts)
    shape = (grid.cells_s(), grid.cells_t())
    tel = RunTelemetry()
    t0 = time.perf_counter()
    if executor.world == 1 and not executor.comm:
        k = np.zeros(shape); l = np.zeros(shape)
        up = np.zeros(shape); lo = np.zeros(shape); diff = np.zeros(shape)
        st = _lib.StkTelemetry()
        d.check(d.lib.stk_run_job(d.h, _lib.ptr(pts.x), _lib.ptr(pts.y),
                                  _lib.ptr(pts.t, C.c_int64), n, int(spec.sims), int(spec.seed),
                                  int(spec.method), _lib.ptr(k), _lib.ptr(l), _lib.ptr(up),
                                  _lib.ptr(lo), _lib.ptr(diff), C.byref(st)))
        tel.pair_comparisons = int(st.candidate_pairs)
        tel.in_threshold_pairs = int(st.in_threshold_pairs)
        tel.exact_path_pairs = int(st.exact_path_pairs)
        tel.device_ms = float(st.total_ms)
        tel.pair_ms = float(st.pair_ms)
        tel.estimation_seconds = time.perf_counter() - t0
        res = RunResult(KSurface(grid, k, SurfaceKind.K), KSurface(grid, l, SurfaceKind.L),
                        theoretical_surface(grid), telemetry=tel)
        if spec.sims > 0:
            res.upper_l = KSurface(grid, up, SurfaceKind.L)
            res.lower_l = KSurface(grid, lo, SurfaceKind.L)
            res.diff_upper = KSurface(grid, diff, SurfaceKind.Diff)
        return res

    if executor.comm:
        # one collective library call: shard + realisation block, exact NCCL
        # exchange and finalize on the device; every rank gets the result
        k = np.zeros(shape); l = np.zeros(shape)
        up = np.zeros(shape); lo = np.zeros(shape); diff = np.zeros(shape)
        st = _lib.StkTelemetry()
        d.check(d.lib.stk_run_job_dist(d.h, _lib.ptr(pts.x), _lib.ptr(pts.y),
                                       _lib.ptr(pts.t, C.c_int64), n, int(spec.sims),
                                       int(spec.seed), int(spec.method), _lib.ptr(k), _lib.ptr(l),
                                       _lib.ptr(up), _lib.ptr(lo), _lib.ptr(diff), C.byref(st)))
        tel.pair_comparisons = int(st.candidate_pairs)
        tel.in_threshold_pairs = int(st.in_threshold_pairs)
        tel.exact_path_pairs = int(st.exact_path_pairs)
        tel.device_ms = float(st.total_ms)
        tel.pair_ms = float(st.pair_ms)
        tel.estimation_seconds = time.perf_counter() - t0
        res = RunResult(KSurface(grid, k, SurfaceKind.K), KSurface(grid, l, SurfaceKind.L),
                        theoretical_surface(grid), telemetry=tel)
        if spec.sims > 0:
            res.upper_l = KSurface(grid, up, SurfaceKind.L)
            res.lower_l = KSurface(grid, lo, SurfaceKind.L)
            res.diff_upper = KSurface(grid, diff, SurfaceKind.Diff)
        return res

    # --- multi-process over a host group: one call per rank (its slice of the
    # observed pattern's pair work + its block of realisations), then the two
    # exact all-reduces.
    r0, r1 = executor.sim_range(spec.sims)
    counts = np.zeros(shape, np.uint64)
    hi = np.zeros(shape, np.uint64)
    lo = np.zeros(shape, np.uint64)
    up = np.full(shape, -np.inf)
    lower = np.full(shape, np.inf)
    st = _lib.StkTelemetry()
    d.check(d.lib.stk_run_job_shard(d.h, _lib.ptr(pts.x), _lib.ptr(pts.y),
                                    _lib.ptr(pts.t, C.c_int64), n, executor.rank, executor.world,
                                    r0, r1, int(spec.seed), int(spec.method),
                                    _lib.ptr(counts, C.c_uint64), _lib.ptr(hi, C.c_uint64),
                                    _lib.ptr(lo, C.c_uint64), _lib.ptr(up), _lib.ptr(lower),
                                    C.byref(st)))
    return _combine_ranks(executor, region, grid, n, spec, counts, hi, lo, up, lower, st, t0, d)


def _combine_ranks(executor, region, grid, n, spec, counts, hi, lo, up, lower, st, t0, d):
    """The exchange step shared by run_job and bench: exact SUM of the observed
    partials, MAX/MIN of the partial envelopes, then finalize on every rank."""
    counts, hi, lo = executor.allreduce_exact(counts, hi, lo)
    k_hat, l_hat = finalize_exact(hi, lo, n, region, grid, d)
    tel = RunTelemetry(pair_comparisons=int(st.candidate_pairs),
                       in_threshold_pairs=int(st.in_threshold_pairs),
                       exact_path_pairs=int(st.exact_path_pairs), device_ms=float(st.total_ms),
                       pair_ms=float(st.pair_ms))
    res = RunResult(k_hat, l_hat, theoretical_surface(grid), telemetry=tel)
    if spec.sims > 0:
        up, lower = executor.allreduce_envelopes(up, lower)
        res.upper_l = KSurface(grid, up, SurfaceKind.L)
        res.lower_l = KSurface(grid, lower, SurfaceKind.L)
        e = l_hat.values
        res.diff_upper = KSurface(grid, np.where(e > up, e - up, 0.0), SurfaceKind.Diff)
    tel.estimation_seconds = time.perf_counter() - t0
    return res
