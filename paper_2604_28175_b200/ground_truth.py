"""Hidden ground-truth slowdown (infersim/oracle.py:55-77) on the device
(strait_gt_slowdown; the same arithmetic the replay engine runs per started
co-runner, csrc/strait_replay_impl.cuh gt_slowdown).  The parameter types
(GroundTruthParams, default_ground_truth) live in config.py."""
from __future__ import annotations

import ctypes as C
from typing import Sequence

import numpy as np
import torch

from . import _device as D
from ._abi import MAX_METRICS
from .config import GroundTruthParams
from .domain import PriorityLevel


class GroundTruth(C.Structure):
    """include/strait.h StraitGroundTruth."""
    _fields_ = [("family", C.c_int32), ("n_metrics", C.c_int32), ("scale", C.c_double), ("base", C.c_double),
                ("offset", C.c_double), ("w_cmp", C.c_double), ("w_mem", C.c_double), ("pf_high", C.c_double),
                ("pf_low", C.c_double), ("w", C.c_double * MAX_METRICS)]


def _struct(p: GroundTruthParams) -> GroundTruth:
    if len(p.weights) > MAX_METRICS:
        raise ValueError(f"at most {MAX_METRICS} metrics")
    g = GroundTruth()
    g.family = 0 if p.family == "exponential" else 1
    g.n_metrics = len(p.weights)
    g.scale, g.base, g.offset = p.scale, p.base, p.offset
    g.w_cmp, g.w_mem = p.self_compute_weight, p.self_memory_weight
    g.pf_high, g.pf_low = p.priority_factor[PriorityLevel.HIGH], p.priority_factor[PriorityLevel.LOW]
    for i, w in enumerate(p.weights):
        g.w[i] = w
    return g


def ground_truth_slowdown_batch(params: GroundTruthParams, colocated, self_compute, self_memory, priority,
                                noise=None) -> np.ndarray:
    """Vectorised oracle.py:55-77: colocated is [n, n_metrics]."""
    co = np.asarray(colocated, dtype=np.float64)
    if co.ndim != 2 or co.shape[1] != len(params.weights):
        raise ValueError(f"aggregate throughput has {co.shape[-1] if co.ndim else 0} metrics, "
                         f"oracle expects {len(params.weights)}")
    n = co.shape[0]
    out = D.empty(max(n, 1))
    t = [D.dev(np.ascontiguousarray(co.T)), D.dev(np.asarray(self_compute, np.float64)),
         D.dev(np.asarray(self_memory, np.float64)), D.dev(np.asarray(priority, np.int8), torch.int8)]
    nz = D.dev(np.asarray(noise, np.float64)) if noise is not None else None
    g = _struct(params)
    D.check(D.lib().strait_gt_slowdown(C.byref(g), D.ptr(t[0]), D.ptr(t[1]), D.ptr(t[2]), D.ptr(t[3]), D.ptr(nz), n,
                                       D.ptr(out), D.stream_handle()))
    return D.host(out)[:n]


def ground_truth_slowdown(params: GroundTruthParams, colocated: Sequence[float], self_compute: float,
                          self_memory: float, priority: PriorityLevel, noise: float = 1.0) -> float:
    """oracle.py:55-77: instantaneous slowdown under the co-located aggregate
    throughput; 1 when the raw effect clamps to zero."""
    if len(colocated) != len(params.weights):
        raise ValueError(f"aggregate throughput has {len(colocated)} metrics, oracle expects {len(params.weights)}")
    return float(ground_truth_slowdown_batch(params, [list(colocated)], [self_compute], [self_memory],
                                             [int(priority)], [noise])[0])
