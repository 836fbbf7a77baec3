"""ctypes mirror of include/strait.h and the loader for the in-tree CUDA
library ``_strait.so``.

There is deliberately no fallback: if the library (or a GPU) is missing the
product path raises ``StraitUnavailable`` instead of computing anything on the
CPU.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# STRAIT_LIB: an alternative build of the same library (diagnostic builds, e.g. `make prof`)
LIB_PATH = os.environ.get("STRAIT_LIB") or os.path.join(_HERE, "_strait.so")

ABI_VERSION = 2  # include/strait.h STRAIT_ABI_VERSION
STRAIT_OK = 0
STRAIT_EINVAL = 1
STRAIT_ERUNTIME = 2
STRAIT_EORDER = 3
STRAIT_ECUDA = 4
MAX_METRICS = 8

PAIR_HAS_SLOT = 1
PAIR_VIOLATE = 2
PAIR_MEET = 4
PAIR_FEASIBLE = 8

_dp = C.POINTER(C.c_double)
_vp = C.c_void_p


class StraitUnavailable(RuntimeError):
    """The CUDA library or device is missing: the product path refuses to run."""


class SimulationOrderError(Exception):
    """A timeline or event was touched with a timestamp moving backwards
    (mirrors infersim.domain.SimulationOrderError, domain.py:47-49)."""


class StraitCudaError(RuntimeError):
    pass


class SweepArgs(C.Structure):
    _fields_ = [
        ("n_metrics", C.c_int32),
        ("n_slots", C.c_int32),
        ("gpus_per_segment", C.c_int32),
        ("concurrency_limit", C.c_int32),
        ("n_segments", C.c_int64),
        ("now", C.c_double),
        ("effect_cap", C.c_double),
        ("use_violate", C.c_int32),
        ("use_meet", C.c_int32),
        ("params", _vp),
        ("cand_contrib", _vp),
        ("cand_self_cmp", _vp),
        ("cand_self_mem", _vp),
        ("cand_total", _vp),
        ("cand_kernel", _vp),
        ("cand_deadline", _vp),
        ("cand_front", _vp),
        ("cand_prio", _vp),
        ("gpu_agg", _vp),
        ("gpu_lp_agg", _vp),
        ("gpu_cap_pct", _vp),
        ("gpu_t_avail", _vp),
        ("gpu_n_running", _vp),
        ("ent_contrib", _vp),
        ("ent_twa", _vp),
        ("ent_self_cmp", _vp),
        ("ent_self_mem", _vp),
        ("ent_t_kernel", _vp),
        ("ent_deadline_abs", _vp),
        ("ent_kstart", _vp),
        ("ent_prio", _vp),
        ("pair_flags", _vp),
        ("pair_latency", _vp),
        ("pair_intf", _vp),
        ("seg_gpu", _vp),
        ("seg_latency", _vp),
        ("seg_intf", _vp),
    ]


class RefitArgs(C.Structure):
    _fields_ = [
        ("n_metrics", C.c_int32),
        ("n_bc", C.c_int32),
        ("n", C.c_int64),
        ("effect_cap", C.c_double),
        ("learning_rate", C.c_double),
        ("beta1", C.c_double),
        ("beta2", C.c_double),
        ("eps", C.c_double),
        ("huber_delta", C.c_double),
        ("state", _vp),
        ("step", _vp),
        ("bc1", _vp),
        ("bc2", _vp),
        ("twa", _vp),
        ("self_cmp", _vp),
        ("self_mem", _vp),
        ("actual", _vp),
        ("prio", _vp),
        ("out_predicted", _vp),
        ("out_residual", _vp),
        ("out_flags", _vp),
    ]


class SweepExpandArgs(C.Structure):
    _fields_ = [("table_stride", C.c_int32), ("pad", C.c_int32), ("thr", _vp), ("self_cmp", _vp),
                ("self_mem", _vp), ("kernel", _vp), ("total", _vp), ("deadline", _vp), ("prio", _vp),
                ("ent_row", _vp), ("cand_row", _vp), ("n_rows", C.c_int64)]


# field groups of SweepArgs, used by exporters
SWEEP_CAND_FIELDS = ("cand_contrib", "cand_self_cmp", "cand_self_mem", "cand_total",
                     "cand_kernel", "cand_deadline", "cand_front", "cand_prio")
SWEEP_PAIR_FIELDS = ("gpu_agg", "gpu_lp_agg", "gpu_cap_pct", "gpu_t_avail", "gpu_n_running")
SWEEP_ENT_FIELDS = ("ent_contrib", "ent_twa", "ent_self_cmp", "ent_self_mem", "ent_t_kernel",
                    "ent_deadline_abs", "ent_kstart", "ent_prio")
SWEEP_OUT_FIELDS = ("pair_flags", "pair_latency", "pair_intf", "seg_gpu", "seg_latency", "seg_intf")
REFIT_SAMPLE_FIELDS = ("twa", "self_cmp", "self_mem", "actual", "prio")

_lib = None
_lock = threading.Lock()


def _declare(lib):
    lib.strait_abi_version.restype = C.c_int
    lib.strait_struct_size.restype = C.c_int64
    lib.strait_struct_size.argtypes = [C.c_int32]
    lib.strait_last_error.restype = C.c_char_p
    lib.strait_kernel_launches.restype = C.c_int64
    lib.strait_predict.restype = C.c_int
    lib.strait_predict.argtypes = [_vp, C.c_int32, C.c_double, _vp, _vp, _vp, _vp, C.c_int64,
                                   _vp, _vp, _vp]
    lib.strait_predict_parts.restype = C.c_int
    lib.strait_predict_parts.argtypes = [_vp, C.c_int32, C.c_double, _vp, _vp, _vp, _vp, C.c_int64,
                                         _vp, _vp, _vp, _vp, _vp]
    lib.strait_last_sweep_path.restype = C.c_int
    lib.strait_kernel_effect.restype = C.c_int
    lib.strait_kernel_effect.argtypes = [_vp, C.c_int32, C.c_double, _vp, C.c_int64, _vp, _vp, _vp]
    lib.strait_twa.restype = C.c_int
    lib.strait_twa.argtypes = [C.c_int32, _vp, _vp, _vp, _vp, _vp, C.c_int64, _vp, _vp]
    lib.strait_estimate_latency.restype = C.c_int
    lib.strait_estimate_latency.argtypes = [_vp, C.c_int32, C.c_double] + [_vp] * 9 + [
        C.c_int64, _vp, _vp, _vp]
    lib.strait_sweep.restype = C.c_int
    lib.strait_sweep.argtypes = [C.POINTER(SweepArgs), _vp]
    lib.strait_refit.restype = C.c_int
    lib.strait_refit.argtypes = [C.POINTER(RefitArgs), _vp]
    lib.strait_round.restype = C.c_int
    lib.strait_round.argtypes = [C.POINTER(SweepArgs), C.POINTER(RefitArgs), _vp]
    lib.strait_math.restype = C.c_int
    lib.strait_math.argtypes = [C.c_int32, _vp, _vp, C.c_int64, _vp, _vp]
    lib.strait_loss_gradient.restype = C.c_int
    lib.strait_loss_gradient.argtypes = [_vp, C.c_int32, C.c_double, C.c_double] + [_vp] * 5 + [C.c_int64] + [_vp] * 5
    lib.strait_adam_step.restype = C.c_int
    lib.strait_adam_step.argtypes = [_vp] * 5 + [C.c_int32] + [C.c_double] * 6 + [_vp]
    lib.strait_huber.restype = C.c_int
    lib.strait_huber.argtypes = [_vp, C.c_double, C.c_int64, _vp, _vp, _vp]
    lib.strait_gt_slowdown.restype = C.c_int
    lib.strait_gt_slowdown.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, C.c_int64, _vp, _vp]
    lib.strait_sweep_expand.restype = C.c_int
    lib.strait_sweep_expand.argtypes = [C.POINTER(SweepExpandArgs), C.POINTER(SweepArgs), _vp]
    if hasattr(lib, "strait_replay"):
        from ._replay_abi import declare_replay

        declare_replay(lib)
    if hasattr(lib, "strait_stream_count"):
        from .devgen import declare

        declare(lib)


def lib():
    """The loaded CUDA library; raises StraitUnavailable if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise StraitUnavailable(
                    f"{LIB_PATH} is not built; run `make` (or __graft_entry__.build())"
                )
            handle = C.CDLL(LIB_PATH)
            _declare(handle)
            if handle.strait_abi_version() != ABI_VERSION:
                raise StraitUnavailable("strait ABI version mismatch")
            _lib = handle
    return _lib


def check(status: int) -> None:
    """Map a C-ABI status code onto the reference's exception types."""
    if status == STRAIT_OK:
        return
    msg = lib().strait_last_error().decode(errors="replace")
    if status == STRAIT_EINVAL:
        raise ValueError(msg)
    if status == STRAIT_ERUNTIME:
        raise RuntimeError(msg)
    if status == STRAIT_EORDER:
        raise SimulationOrderError(msg)
    raise StraitCudaError(msg)


def check_code(status: int, context: str = "") -> None:
    """Raise the reference's exception for a per-replay/per-item status code."""
    if status == STRAIT_OK:
        return
    msg = f"{context}: status {status}"
    if status == STRAIT_EINVAL:
        raise ValueError(msg)
    if status == STRAIT_ERUNTIME:
        raise RuntimeError(msg)
    if status == STRAIT_EORDER:
        raise SimulationOrderError(msg)
    raise StraitCudaError(msg)
