"""ctypes mirror of include/strait_replay.h."""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._abi import MAX_METRICS

_vp = C.c_void_p

RC = dict(ERROR=0, BATCHES=1, COMPLETED=2, PASSES=3, CAP_ROWS=4, EVENTS=5, HP_ARR=6, LP_ARR=7, HP_VIOL=8,
          LP_VIOL=9, HP_DROP=10, LP_DROP=11, RESOLVED=12, TRACE=13)
RC_N = 16


class ReplayModels(C.Structure):
    _fields_ = [("n_models", C.c_int32), ("n_metrics", C.c_int32), ("stride", C.c_int32), ("pad", C.c_int32),
                ("max_batch", _vp), ("prio", _vp), ("deadline", _vp), ("timeout", _vp), ("total", _vp),
                ("transfer", _vp), ("kernel", _vp), ("self_cmp", _vp), ("self_mem", _vp), ("throughput", _vp)]


class ReplayConfig(C.Structure):
    _fields_ = [("n_gpus", C.c_int32), ("concurrency_limit", C.c_int32), ("use_priority_order", C.c_int32),
                ("use_meet", C.c_int32), ("use_violate", C.c_int32), ("gt_family", C.c_int32),
                ("has_noise", C.c_int32), ("policy", C.c_int32), ("refit_frozen", C.c_int32),
                ("reserved0", C.c_int32),
                ("effect_cap", C.c_double), ("learning_rate", C.c_double), ("beta1", C.c_double),
                ("beta2", C.c_double), ("eps", C.c_double), ("huber_delta", C.c_double),
                ("gt_scale", C.c_double), ("gt_base", C.c_double), ("gt_offset", C.c_double),
                ("gt_w_cmp", C.c_double), ("gt_w_mem", C.c_double), ("gt_pf_high", C.c_double),
                ("gt_pf_low", C.c_double), ("gt_w", C.c_double * MAX_METRICS),
                ("aimd_floor", C.c_double), ("aimd_ceiling", C.c_double), ("aimd_increase", C.c_double),
                ("aimd_interval", C.c_double), ("static_cap", C.c_int32), ("reactive_default", C.c_int32),
                ("reactive_min", C.c_int32), ("reactive_hp_bound", C.c_int32), ("reactive_period", C.c_double)]

POLICY_CODES = {"predictive": 0, "temporal": 1, "static": 2, "reactive": 3}


ARG_ARRAYS = ["cfg", "req_off", "arr_time", "arr_model", "model_req", "mr_off", "noise", "bc1", "bc2",
              "pred_state", "pred_step", "req_status", "req_violated", "req_completion", "req_batch",
              "dec_time", "dec_pass", "dec_model", "dec_size", "dec_gpu", "dec_est_latency", "dec_intf",
              "b_front", "b_transfer_start", "b_transfer_end", "b_kernel_start", "b_kernel_end", "b_completion",
              "b_work", "b_done_order", "fb_predicted", "fb_actual", "fb_residual", "fb_flags",
              "cap_time", "cap_gpu", "cap_pct", "counters", "order", "trace"]


class ReplayArgs(C.Structure):
    _fields_ = [("n_replays", C.c_int32), ("cap_rows_max", C.c_int32), ("n_bc", C.c_int32),
                ("max_gpus", C.c_int32), ("max_concurrency", C.c_int32), ("trace_max", C.c_int32),
                ("policies", C.c_int32), ("uniform", C.c_int32),
                ("models", ReplayModels)] + [(k, _vp) for k in ARG_ARRAYS]


# StraitTraceRec and the STRAIT_TR_* event codes
TRACE_DTYPE = np.dtype([("time", "<f8"), ("x", "<f8", (3,)), ("request", "<i8"), ("batch", "<i4"),
                        ("gpu", "<i2"), ("event", "i1"), ("size", "i1")])
assert TRACE_DTYPE.itemsize == 48
TR = dict(ARRIVAL=0, SUBMIT=1, DROP=2, KSTART=3, KDONE=4, TICK=5, RESET=6, SEGMENT=7)

MS_N = 5
METRIC_ARRAYS = ["window_ms", "req_off", "arr_time", "arr_model", "model_prio", "req_status", "req_violated",
                 "req_completion", "counters", "dec_model", "dec_size", "dec_est_latency", "b_front",
                 "b_kernel_start", "b_kernel_end", "b_completion", "fb_predicted", "fb_actual", "kernel_table"]
METRIC_OUTPUTS = ["class_counts", "partial", "pct", "series_count", "goodput", "goodput_len", "intf_error",
                  "latency_error", "kernel_overhead"]


class MetricsArgs(C.Structure):
    _fields_ = ([("n_replays", C.c_int32), ("max_windows", C.c_int32)] + [(k, _vp) for k in METRIC_ARRAYS]
                + [("table_stride", C.c_int32), ("pad", C.c_int32)] + [(k, _vp) for k in METRIC_OUTPUTS])


def declare_replay(lib):
    lib.strait_replay.restype = C.c_int
    lib.strait_replay.argtypes = [C.POINTER(ReplayArgs), _vp]
    lib.strait_replay_metrics.restype = C.c_int
    lib.strait_replay_metrics.argtypes = [C.POINTER(MetricsArgs), _vp]
    lib.strait_replay_smem_bytes.restype = C.c_int64
    lib.strait_replay_smem_bytes.argtypes = [C.c_int32] * 4
