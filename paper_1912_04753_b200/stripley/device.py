"""Device contexts: one ``stk_ctx`` (one CUDA device, one stream) per device.

A context caches the region and grid it was last configured with, so repeated
calls on the same study setup upload nothing but points.
"""
from __future__ import annotations

import ctypes as C
import threading

import numpy as np

from .. import _lib


class Device:
    def __init__(self, device: int = 0):
        lib = _lib.load()
        h = C.c_void_p()
        rc = lib.stk_create(C.byref(h), int(device))
        if rc != 0 or not h.value:
            raise RuntimeError(
                f"stk_create(device={device}) failed: no usable CUDA device "
                "(the B200 path has no CPU fallback)")
        self.lib = lib
        self.h = h
        self.index = int(device)
        self._region_key = None
        self._grid_key = None

    # -- errors -----------------------------------------------------------
    def check(self, rc: int):
        if rc == _lib.STK_OK:
            return
        msg = self.lib.stk_last_error(self.h).decode()
        if rc == _lib.STK_EINVAL:
            raise ValueError(msg)
        if rc == _lib.STK_EUNSUPPORTED:
            raise NotImplementedError(msg)
        raise _lib.StkError(f"stk error {rc}: {msg}")

    # -- configuration ----------------------------------------------------
    def configure(self, region, grid=None, options=None):
        rk = region.key()
        if rk != self._region_key:
            ring = np.ascontiguousarray(region.boundary().reshape(-1))
            self.check(self.lib.stk_set_region(self.h, _lib.ptr(ring), len(ring) // 2,
                                               region.period_start(), region.period_end()))
            self._region_key = rk
        if grid is not None:
            gk = grid.key()
            if gk != self._grid_key:
                s = _lib.f64(grid.s_values)
                t = _lib.i64(grid.t_values)
                self.check(self.lib.stk_set_grid(self.h, _lib.ptr(s), len(s),
                                                 _lib.ptr(t, C.c_int64), len(t)))
                self._grid_key = gk
        if options is not None:
            self.check(self.lib.stk_set_options(self.h, int(options.use_index),
                                                int(options.use_cache),
                                                float(options.coord_tolerance),
                                                float(options.dist_tolerance)))

    def stream_handle(self) -> int:
        return int(self.lib.stk_stream(self.h) or 0)

    def set_memory_budget(self, nbytes: int):
        self.check(self.lib.stk_set_memory_budget(self.h, int(nbytes)))

    def set_rng(self, rng: str):
        """Realisation generator: "mt19937_64" (default; the reference's stream,
        bit-exact) or "philox" (opt-in Philox4x32-10, statistical parity)."""
        code = {"mt19937_64": _lib.RNG_MT19937_64, "philox": _lib.RNG_PHILOX}[rng]
        self.check(self.lib.stk_set_rng(self.h, code))

    def philox4x32(self, ctr, key):
        """Raw device Philox4x32-10 blocks (known-answer tests)."""
        ctr = np.ascontiguousarray(ctr, np.uint32).reshape(-1, 4)
        key = np.ascontiguousarray(key, np.uint32).reshape(-1, 2)
        out = np.zeros_like(ctr)
        u32p = C.POINTER(C.c_uint32)
        self.check(self.lib.stk_philox4x32(self.h, ctr.ctypes.data_as(u32p),
                                           key.ctypes.data_as(u32p), len(ctr),
                                           out.ctypes.data_as(u32p)))
        return out

    # -- multi-GPU: NCCL communicator inside the library ---------------------
    def comm_init(self, unique_id: bytes, nranks: int, rank: int):
        """stk_comm_init: join the communicator of ``unique_id`` (from
        :func:`nccl_unique_id` on rank 0) as ``rank`` of ``nranks``."""
        if len(unique_id) != _lib.NCCL_ID_BYTES:
            raise ValueError("NCCL unique id must be 128 bytes")
        self.check(self.lib.stk_comm_init(self.h, bytes(unique_id), int(nranks), int(rank)))

    def comm_destroy(self):
        self.check(self.lib.stk_comm_destroy(self.h))

    def comm_rank(self):
        """(rank, nranks) of the context's communicator, or None without one."""
        r, n = C.c_int(), C.c_int()
        rc = self.lib.stk_comm_rank(self.h, C.byref(r), C.byref(n))
        return (r.value, n.value) if rc == _lib.STK_OK else None

    def fp64_peak(self) -> float:
        v = C.c_double()
        self.check(self.lib.stk_measure_fp64_peak(self.h, C.byref(v)))
        return v.value

    def close(self):
        if self.h is not None and self.h.value:
            self.lib.stk_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    """stk_comm_unique_id (ncclGetUniqueId through the library)."""
    lib = _lib.load()
    buf = C.create_string_buffer(_lib.NCCL_ID_BYTES)
    rc = lib.stk_comm_unique_id(buf)
    if rc != _lib.STK_OK:
        raise _lib.StkError("stk_comm_unique_id failed: NCCL unavailable")
    return buf.raw


_devices: dict[int, Device] = {}
_lock = threading.Lock()


def get(device: int | None = None) -> Device:
    """The shared context of ``device`` (default: current torch device or 0)."""
    if device is None:
        device = 0
        try:
            import torch

            if torch.cuda.is_available():
                device = torch.cuda.current_device()
        except Exception:
            pass
    with _lock:
        d = _devices.get(device)
        if d is None:
            d = Device(device)
            _devices[device] = d
        return d
