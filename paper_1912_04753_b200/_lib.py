"""ctypes binding of ``libstk.so`` (the C ABI declared in ``include/stk.h``).

The library is built in-tree by ``__graft_entry__.build()`` /
``paper_1912_04753_b200.build.build_library()``.  There is no CPU fallback:
if the library or a CUDA device is missing, every hot-path call raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("STK_LIB_PATH") or os.path.join(HERE, "libstk.so")

STK_OK, STK_EINVAL, STK_EUNSUPPORTED, STK_ECUDA, STK_ESTATE, STK_ENCCL = 0, 1, 2, 3, 4, 5
NCCL_ID_BYTES = 128
RNG_MT19937_64, RNG_PHILOX = 0, 1
METHOD_CSR, METHOD_BOOTSTRAP, METHOD_PERMUTATION = 0, 1, 2


class StkTelemetry(C.Structure):
    _fields_ = [
        ("in_threshold_pairs", C.c_uint64),
        ("candidate_pairs", C.c_uint64),
        ("exact_path_pairs", C.c_uint64),
        ("patterns", C.c_uint64),
        ("gen_ms", C.c_double),
        ("grid_ms", C.c_double),
        ("pair_ms", C.c_double),
        ("finalize_ms", C.c_double),
        ("total_ms", C.c_double),
        ("kernel_launches", C.c_uint64),
        ("arc_pairs", C.c_uint64),
        ("batches", C.c_uint64),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


# Every symbol include/stk.h declares (checked by tests/test_abi_cpu.py).
EXPORTED = [
    "stk_check_region", "stk_check_grid", "stk_create", "stk_destroy", "stk_last_error",
    "stk_version", "stk_stream", "stk_set_memory_budget", "stk_set_region", "stk_set_grid",
    "stk_set_options", "stk_estimate_surface", "stk_pair_histogram", "stk_finalize",
    "stk_simulate", "stk_run_job", "stk_run_job_device", "stk_generate_cstr",
    "stk_spatial_weights", "stk_measure_fp64_peak", "stk_run_job_shard",
    "stk_run_job_shard_device", "stk_generate", "stk_comm_unique_id", "stk_comm_init",
    "stk_comm_destroy", "stk_comm_rank", "stk_run_job_dist", "stk_run_job_dist_device",
    "stk_task_histogram", "stk_set_rng", "stk_philox4x32",
]

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int64)
_up = C.POINTER(C.c_uint64)
_vp = C.c_void_p
_u64, _u32, _i64 = C.c_uint64, C.c_uint32, C.c_int64
_tp = C.POINTER(StkTelemetry)

_SIGS = {
    "stk_check_region": (C.c_int, [_dp, _u32, _i64, _i64, _dp, _ip, C.c_char_p, C.c_size_t]),
    "stk_check_grid": (C.c_int, [_dp, _u32, _ip, _u32, C.c_char_p, C.c_size_t]),
    "stk_create": (C.c_int, [C.POINTER(_vp), C.c_int]),
    "stk_destroy": (None, [_vp]),
    "stk_last_error": (C.c_char_p, [_vp]),
    "stk_version": (C.c_char_p, []),
    "stk_stream": (_vp, [_vp]),
    "stk_set_memory_budget": (C.c_int, [_vp, _u64]),
    "stk_set_region": (C.c_int, [_vp, _dp, _u32, _i64, _i64]),
    "stk_set_grid": (C.c_int, [_vp, _dp, _u32, _ip, _u32]),
    "stk_set_options": (C.c_int, [_vp, C.c_int, C.c_int, C.c_double, C.c_double]),
    "stk_estimate_surface": (C.c_int, [_vp, _dp, _dp, _ip, _u64, _dp, _tp]),
    "stk_pair_histogram": (C.c_int, [_vp, _dp, _dp, _ip, _u64, _u32, _u32, _up, _up, _up, _dp, _tp]),
    "stk_finalize": (C.c_int, [_vp, _u64, _up, _up, _dp, _dp]),
    "stk_simulate": (C.c_int, [_vp, _dp, _dp, _ip, _u64, C.c_int, _u64, _u32, _u32, _dp, _dp, _dp, _tp]),
    "stk_run_job": (C.c_int, [_vp, _dp, _dp, _ip, _u64, _u32, _u64, C.c_int, _dp, _dp, _dp, _dp, _dp, _tp]),
    "stk_run_job_device": (C.c_int, [_vp, _vp, _vp, _vp, _u64, _u32, _u64, C.c_int, _dp, _dp, _dp, _dp, _dp, _tp]),
    "stk_run_job_shard": (C.c_int, [_vp, _dp, _dp, _ip, _u64, _u32, _u32, _u32, _u32, _u64, C.c_int, _up, _up, _up, _dp, _dp, _tp]),
    "stk_run_job_shard_device": (C.c_int, [_vp, _vp, _vp, _vp, _u64, _u32, _u32, _u32, _u32, _u64, C.c_int, _up, _up, _up, _dp, _dp, _tp]),
    "stk_generate_cstr": (C.c_int, [_vp, _u64, _u64, _dp, _dp, _ip]),
    "stk_generate": (C.c_int, [_vp, C.c_int, _u64, _dp, _dp, _ip, _u64, _dp, _dp, _ip]),
    "stk_spatial_weights": (C.c_int, [_vp, _dp, _dp, _dp, _u64, _dp]),
    "stk_measure_fp64_peak": (C.c_int, [_vp, _dp]),
    "stk_comm_unique_id": (C.c_int, [C.c_char_p]),
    "stk_comm_init": (C.c_int, [_vp, C.c_char_p, C.c_int, C.c_int]),
    "stk_comm_destroy": (C.c_int, [_vp]),
    "stk_comm_rank": (C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "stk_run_job_dist": (C.c_int, [_vp, _dp, _dp, _ip, _u64, _u32, _u64, C.c_int, _dp, _dp, _dp, _dp, _dp, _tp]),
    "stk_run_job_dist_device": (C.c_int, [_vp, _vp, _vp, _vp, _u64, _u32, _u64, C.c_int, _dp, _dp, _dp, _dp, _dp, _tp]),
    "stk_set_rng": (C.c_int, [_vp, C.c_int]),
    "stk_philox4x32": (C.c_int, [_vp, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), _u32, C.POINTER(C.c_uint32)]),
    "stk_task_histogram": (C.c_int, [_vp, _dp, _dp, _ip, C.POINTER(C.c_uint32), _u64, _dp, _dp, _ip, C.POINTER(C.c_uint32), _dp, _ip, _u64, _dp, _up, _up]),
}

_lib = None


class StkError(RuntimeError):
    pass


def load():
    """Load libstk.so (raises OSError loudly when it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise OSError(
                f"{LIB_PATH} missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                " (the B200 path has no CPU fallback)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _lib = lib
    return _lib


def ptr(a, ctype=C.c_double):
    """ctypes pointer to a C-contiguous numpy array (or NULL for None)."""
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.POINTER(ctype))


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)
