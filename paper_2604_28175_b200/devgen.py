"""On-device generation of a replay batch's arrival and noise streams
(include/strait_replay.h "On-device workload generation", csrc/strait_rng.cuh):
the same numpy 2.3 streams the host path draws (workload.py:19-152,
simulation.py:163,309-311), produced on the GPU — draw for draw identical —
so 100M-request replays need no host RNG, argsort or H2D of the streams.

Only the stream *descriptions* are built on the host: one spec per numpy
Generator (a model's Poisson arrivals, one trace minute, a uniform stream, a
replay's batch noise).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _device as D
from .workload import MINUTE_MS, read_trace_csv

POISSON, UNIFORM, NOISE = 1, 2, 3
NOISE_STREAM = 1_000_003  # simulation.py:163


class StreamSpec(C.Structure):
    _fields_ = [("entropy", C.c_uint64 * 3), ("n_entropy", C.c_int32), ("mode", C.c_int32),
                ("rate_per_s", C.c_double), ("span_ms", C.c_double), ("offset_ms", C.c_double),
                ("sigma", C.c_double), ("n_draws", C.c_int64)]


def declare(lib):
    vp = C.c_void_p
    lib.strait_stream_count.argtypes = [vp, C.c_int64, vp, vp]
    lib.strait_stream_fill.argtypes = [vp, C.c_int64, vp, vp, vp]
    lib.strait_arrival_order.argtypes = [C.c_int32, C.c_int32, vp, vp, vp, vp, vp, vp]
    lib.strait_rng_draws.argtypes = [vp, C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_int64, vp, vp]
    for f in ("strait_stream_count", "strait_stream_fill", "strait_arrival_order", "strait_rng_draws"):
        getattr(lib, f).restype = C.c_int


def _spec(entropy, mode, rate=0.0, span=0.0, offset=0.0, sigma=0.0, n_draws=0) -> StreamSpec:
    s = StreamSpec()
    for i, e in enumerate(entropy):
        if not 0 <= int(e) < 2 ** 64:
            raise ValueError("stream entropy words must be in [0, 2**64)")
        s.entropy[i] = int(e)
    s.n_entropy, s.mode = len(entropy), mode
    s.rate_per_s, s.span_ms, s.offset_ms, s.sigma, s.n_draws = rate, span, offset, sigma, n_draws
    return s


def model_streams(workload, seed: int, model_ids) -> list[list[StreamSpec]]:
    """Per table model (model_ids order), the specs of its arrival streams in
    output order, seeded as WorkloadSpec.generate seeds them."""
    names = sorted(workload.models)
    out = []
    for mid in model_ids:
        specs = []
        if mid in workload.models:
            idx = names.index(mid)
            w = workload.models[mid]
            dur = workload.duration_ms
            if w.mode == "poisson":
                if w.rate_per_s < 0:
                    raise ValueError(f"rate must be non-negative, got {w.rate_per_s}")
                specs.append(_spec([seed, idx], POISSON, w.rate_per_s, dur))
            elif w.mode == "uniform":
                if w.rate_per_s < 0:
                    raise ValueError(f"rate must be positive, got {w.rate_per_s}")
                if w.rate_per_s > 0:
                    specs.append(_spec([seed, idx], UNIFORM, w.rate_per_s, dur))
            elif w.mode == "trace":  # workload.py:75-104: one Poisson stream per minute
                if w.scale <= 0:
                    raise ValueError(f"scale must be positive, got {w.scale}")
                table = w.trace_table if w.trace_table is not None else read_trace_csv(w.trace_file)
                if w.function_id not in table:
                    raise KeyError(f"function {w.function_id!r} not in trace")
                minutes = table[w.function_id]
                for minute in sorted(minutes):
                    start = minute * MINUTE_MS
                    if start >= dur:
                        break
                    rate = minutes[minute] * w.scale / 60.0
                    span = min(MINUTE_MS, dur - start)
                    specs.append(_spec([seed, idx, minute], POISSON, rate, span, start))
            else:
                raise ValueError(f"unknown workload mode {w.mode!r}")
        out.append(specs)
    return out


def _specs_dev(specs):
    arr = (StreamSpec * max(1, len(specs)))(*specs)
    return D.dev(np.frombuffer(bytes(arr), dtype=np.uint8), torch.uint8)


def generate(items, model_ids, stream=None) -> dict:
    """items: [(workload, seed, noise_sigma)] per replay.  Returns device
    arrays arr_time / arr_model / model_req / noise and host req_off / mr_off."""
    lib = D.lib()
    st = D.stream_handle(stream)
    M = len(model_ids)
    per = [model_streams(w, seed, model_ids) for w, seed, _ in items]
    flat = [s for rep in per for m in rep for s in m]
    dspecs = _specs_dev(flat)
    counts = D.empty(max(1, len(flat)), torch.int64)
    D.check(lib.strait_stream_count(D.ptr(dspecs), len(flat), D.ptr(counts), st))
    cnt = D.host(counts)[:len(flat)]
    offs = np.zeros(len(flat), dtype=np.int64)
    if len(flat):
        offs[1:] = np.cumsum(cnt)[:-1]
    # (replay, model) counts -> model-major offsets
    seg = np.zeros(len(items) * M, dtype=np.int64)
    i = 0
    for r, rep in enumerate(per):
        for m, ms in enumerate(rep):
            seg[r * M + m] = cnt[i:i + len(ms)].sum()
            i += len(ms)
    mr_off = np.concatenate([[0], np.cumsum(seg)]).astype(np.int64)
    N = int(mr_off[-1])
    if N >= 2 ** 31:
        raise ValueError("more than 2**31 requests in one replay batch")
    mm = D.empty(max(1, N))
    D.check(lib.strait_stream_fill(D.ptr(dspecs), len(flat), D.ptr(D.dev(offs, torch.int64)), D.ptr(mm), st))
    arr_time, arr_model = D.empty(max(1, N)), D.empty(max(1, N), torch.int16)
    model_req = D.empty(max(1, N), torch.int32)
    dmr = D.dev(mr_off, torch.int64)
    D.check(lib.strait_arrival_order(len(items), M, D.ptr(dmr), D.ptr(mm), D.ptr(arr_time), D.ptr(arr_model),
                                     D.ptr(model_req), st))
    req_off = mr_off[::M].copy()
    # batch noise: N_r draws per replay (an upper bound on its batches)
    noise = torch.ones(max(1, N), dtype=torch.float64, device=arr_time.device)
    nspecs, noffs = [], []
    for r, (_, seed, sigma) in enumerate(items):
        n_r = int(req_off[r + 1] - req_off[r])
        if sigma > 0 and n_r:
            nspecs.append(_spec([seed, NOISE_STREAM], NOISE, sigma=sigma, n_draws=n_r))
            noffs.append(int(req_off[r]))
    if nspecs:
        dn = _specs_dev(nspecs)
        D.check(lib.strait_stream_fill(D.ptr(dn), len(nspecs), D.ptr(D.dev(np.array(noffs), torch.int64)),
                                       D.ptr(noise), st))
    return {"arr_time": arr_time, "arr_model": arr_model, "model_req": model_req, "noise": noise,
            "req_off": req_off, "mr_off": mr_off, "N": N}


def rng_draws(entropy, kind: int, n: int, loc: float = 0.0, scale: float = 1.0) -> np.ndarray:
    """One numpy Generator stream on the device (kind 0 exponential, 1 normal, 2 raw bits)."""
    ent = D.dev(np.asarray(entropy, dtype=np.uint64).view(np.int64), torch.int64)
    out = D.empty(max(1, n))
    D.check(D.lib().strait_rng_draws(D.ptr(ent), len(entropy), kind, loc, scale, n, D.ptr(out), D.stream_handle()))
    return D.host(out)[:n]
