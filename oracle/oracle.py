"""CPU ORACLE wrapper — test infrastructure only.

Loads oracle/build/libstrait_oracle.so (the plain-C restatement of the
reference hot path, oracle/strait_oracle.c; build with ``make oracle``) and
exposes numpy-in/numpy-out entry points.  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference leg may import this module; the
product package never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2604_28175_b200._abi import REFIT_SAMPLE_FIELDS, SWEEP_OUT_FIELDS, RefitArgs, SweepArgs
from paper_2604_28175_b200.sweep import INPUT_FIELDS

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(_HERE, "build", "libstrait_oracle.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise RuntimeError(f"{LIB} missing: run `make oracle`")
        _lib = C.CDLL(LIB)
        vp = C.c_void_p
        _lib.oracle_predict.argtypes = [vp, C.c_int32, C.c_double, vp, vp, vp, vp, C.c_int64, vp, vp]
        _lib.oracle_estimate_latency.argtypes = [vp, C.c_int32, C.c_double] + [vp] * 9 + [C.c_int64, vp, vp]
        _lib.oracle_sweep.argtypes = [C.POINTER(SweepArgs), C.c_int, C.c_int64, C.c_int64]
        _lib.oracle_refit.argtypes = [C.POINTER(RefitArgs)]
        from paper_2604_28175_b200._replay_abi import ReplayArgs

        _lib.oracle_replay.argtypes = [C.POINTER(ReplayArgs), C.c_int]
        _lib.oracle_replay.restype = C.c_int
        _lib.oracle_exp.argtypes = [vp, vp, C.c_int64]
        _lib.oracle_exp.restype = None
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def predict(P, cap, coloc_mn, cmp_, mem, prio):
    """coloc_mn: metric-major [nm, n] -> (intf[n], saturated[n])."""
    P = _f64(P)
    A = _f64(coloc_mn)
    nm, n = A.shape
    cmp_, mem = _f64(np.broadcast_to(cmp_, (n,))), _f64(np.broadcast_to(mem, (n,)))
    pr = np.ascontiguousarray(np.broadcast_to(prio, (n,)), dtype=np.int8)
    out = np.empty(n)
    sat = np.empty(n, dtype=np.uint8)
    lib().oracle_predict(_p(P), nm, cap, _p(A), _p(cmp_), _p(mem), _p(pr), n, _p(out), _p(sat))
    return out, sat.astype(bool)


def estimate_latency(P, cap, assumed_mn, cmp_, mem, prio, total, kernel, t_avail, front, now):
    P = _f64(P)
    A = _f64(assumed_mn)
    nm, n = A.shape
    f = [_f64(np.broadcast_to(v, (n,))) for v in (cmp_, mem)]
    pr = np.ascontiguousarray(np.broadcast_to(prio, (n,)), dtype=np.int8)
    g = [_f64(np.broadcast_to(v, (n,))) for v in (total, kernel, t_avail, front, now)]
    lat, intf = np.empty(n), np.empty(n)
    lib().oracle_estimate_latency(_p(P), nm, cap, _p(A), _p(f[0]), _p(f[1]), _p(pr), *[_p(x) for x in g], n,
                                  _p(lat), _p(intf))
    return lat, intf


def sweep(soa, P, cap=50.0, use_violate=True, use_meet=True, threads=1, seg_range=None):
    """Reference check_violate/check_meet/best_for over a host SoA."""
    P = _f64(P)
    arrays = {}
    for k in INPUT_FIELDS:
        dt = np.int8 if k in ("cand_prio", "gpu_n_running", "ent_prio") else np.float64
        arrays[k] = np.ascontiguousarray(soa.arrays[k], dtype=dt)
    out = {
        "pair_flags": np.zeros(soa.n_pairs, np.uint8),
        "pair_latency": np.full(soa.n_pairs, np.nan),
        "pair_intf": np.full(soa.n_pairs, np.nan),
        "seg_gpu": np.full(soa.n_segments, -2, np.int32),
        "seg_latency": np.full(soa.n_segments, np.nan),
        "seg_intf": np.full(soa.n_segments, np.nan),
    }
    a = SweepArgs()
    a.n_metrics, a.n_slots, a.gpus_per_segment = soa.n_metrics, soa.n_slots, soa.gpus_per_segment
    a.concurrency_limit, a.n_segments, a.now = soa.concurrency_limit, soa.n_segments, float(soa.now)
    a.effect_cap, a.use_violate, a.use_meet = float(cap), int(use_violate), int(use_meet)
    a.params = _p(P)
    for k, v in arrays.items():
        setattr(a, k, _p(v))
    for k in SWEEP_OUT_FIELDS:
        setattr(a, k, _p(out[k]))
    s0, s1 = seg_range if seg_range is not None else (0, -1)
    lib().oracle_sweep(C.byref(a), int(threads), int(s0), int(s1))
    return out


def refit(state, step, samples, *, nm, cap=50.0, lr=0.0075, beta1=0.7, beta2=0.9, eps=1e-8, delta=0.5):
    """Sequential reference update over samples (dict of SoA arrays).
    Returns (state, step, predicted, residual, flags)."""
    state = _f64(state).copy()
    stepa = np.array([step], dtype=np.int64)
    n = len(samples["actual"])
    arr = {k: (np.ascontiguousarray(samples[k], dtype=np.int8) if k == "prio" else _f64(samples[k]))
           for k in REFIT_SAMPLE_FIELDS}
    pred, res, flags = np.empty(n), np.empty(n), np.empty(n, np.uint8)
    a = RefitArgs()
    a.n_metrics, a.n_bc, a.n = nm, 0, n
    a.effect_cap, a.learning_rate, a.beta1, a.beta2, a.eps, a.huber_delta = cap, lr, beta1, beta2, eps, delta
    a.state, a.step = _p(state), _p(stepa)
    for k in REFIT_SAMPLE_FIELDS:
        setattr(a, k, _p(arr[k]))
    a.out_predicted, a.out_residual, a.out_flags = _p(pred), _p(res), _p(flags)
    lib().oracle_refit(C.byref(a))
    return state, int(stepa[0]), pred, res, flags


def exp(z):
    """glibc exp elementwise (the reference's math.exp)."""
    z = _f64(z)
    out = np.empty_like(z)
    lib().oracle_exp(_p(z), _p(out), z.size)
    return out


def replay(batch, threads=1):
    """Reference discrete-event replay (oracle/strait_replay_oracle.c) of a
    paper_2604_28175_b200.replay.ReplayBatch on host buffers."""
    from paper_2604_28175_b200.replay import ReplayResult

    inputs = batch.host_inputs()
    if "noise_z" in inputs:  # host-drawn normals -> math.exp(z) with glibc (simulation.py:309-311)
        inputs["noise"] = exp(inputs.pop("noise_z"))
    inputs["pred_state"] = inputs["pred_state"].copy()
    inputs["pred_step"] = inputs["pred_step"].copy()
    outputs = batch.alloc_outputs(device=False)

    def ptr(a):
        return C.addressof(a) if isinstance(a, C.Array) else a.ctypes.data

    args = batch.args(inputs, outputs, ptr)
    lib().oracle_replay(C.byref(args), int(threads))
    outputs["pred_state"] = inputs["pred_state"]
    outputs["pred_step"] = inputs["pred_step"]
    return ReplayResult(batch, outputs)
