"""Structure-of-arrays candidate sweep: the batched form of
``PredictivePolicy.best_for`` (scheduler.py:263-280) over independent
(candidate, GPU, co-runner) snapshots, plus the fused sweep+refit round.

A ``SweepSoA`` holds host (numpy) or device (torch) arrays named after the
fields of ``StraitSweepArgs`` (include/strait.h).  Per-metric fields are
metric-major ``[n_metrics, n]``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as D
from ._abi import (SWEEP_CAND_FIELDS, SWEEP_ENT_FIELDS, SWEEP_OUT_FIELDS, SWEEP_PAIR_FIELDS, RefitArgs,
                   SweepArgs)

INT8_FIELDS = {"cand_prio", "gpu_n_running", "ent_prio"}
METRIC_FIELDS = {"cand_contrib", "gpu_agg", "gpu_lp_agg", "ent_contrib", "ent_twa"}
OUT_DTYPES = {"pair_flags": torch.uint8, "pair_latency": torch.float64, "pair_intf": torch.float64,
              "seg_gpu": torch.int32, "seg_latency": torch.float64, "seg_intf": torch.float64}
INPUT_FIELDS = SWEEP_CAND_FIELDS + SWEEP_PAIR_FIELDS + SWEEP_ENT_FIELDS
# packed device blocks (row order = the kernel's stage layout)
ENT_BLOCK, PAIR_BLOCK = "ent", "pair"
ENT_ROWS = ("ent_contrib", "ent_twa", "ent_self_cmp", "ent_self_mem", "ent_t_kernel", "ent_deadline_abs",
            "ent_kstart")
PAIR_ROWS = ("gpu_agg", "gpu_lp_agg", "gpu_cap_pct", "gpu_t_avail")


@dataclass
class SweepSoA:
    n_metrics: int
    n_slots: int
    gpus_per_segment: int
    concurrency_limit: int
    n_segments: int
    now: float
    arrays: dict = field(default_factory=dict)

    @property
    def n_pairs(self) -> int:
        return self.n_segments * self.gpus_per_segment

    @property
    def n_triples(self) -> int:
        return self.n_pairs * self.n_slots

    def like(self, arrays: dict) -> "SweepSoA":
        return SweepSoA(self.n_metrics, self.n_slots, self.gpus_per_segment, self.concurrency_limit,
                        self.n_segments, self.now, arrays)

    def to_device(self) -> "SweepSoA":
        """Device copy in the PACKED layout: the triple fields are rows of one
        [2*nm+5, T] block and the pair fields rows of one [2*nm+2, P] block, so the
        sweep can move a tile with two 2-D TMA tensor copies."""
        out = {}
        nm = self.n_metrics
        for block, fields, n in ((ENT_BLOCK, ENT_ROWS, self.n_triples), (PAIR_BLOCK, PAIR_ROWS, self.n_pairs)):
            rows = sum(nm if f in METRIC_FIELDS else 1 for f in fields)
            buf = D.empty((rows, n))
            r = 0
            for f in fields:
                k = nm if f in METRIC_FIELDS else 1
                view = buf[r:r + k] if k > 1 or f in METRIC_FIELDS else buf[r]
                view.copy_(torch.from_numpy(np.ascontiguousarray(self.arrays[f], dtype=np.float64))
                           if not isinstance(self.arrays[f], torch.Tensor) else self.arrays[f])
                out[f] = view
                r += k
        for k in INPUT_FIELDS:
            if k not in out:
                dt = torch.int8 if k in INT8_FIELDS else torch.float64
                out[k] = D.dev(self.arrays[k], dt)
        return self.like(out)

    def input_bytes(self) -> int:
        """Algorithmic input bytes of one sweep over this SoA."""
        return int(sum(np.asarray(self.arrays[k]).nbytes if not isinstance(self.arrays[k], torch.Tensor)
                       else self.arrays[k].numel() * self.arrays[k].element_size() for k in INPUT_FIELDS))

    def slice_segments(self, s0: int, s1: int) -> "SweepSoA":
        """Host sub-SoA of segments [s0, s1) (contiguous in every field)."""
        G, Cs = self.gpus_per_segment, self.n_slots
        cut = {}
        for k in INPUT_FIELDS:
            a = self.arrays[k]
            if k.startswith("cand"):
                lo, hi = s0, s1
            elif k.startswith("gpu"):
                lo, hi = s0 * G, s1 * G
            else:
                lo, hi = s0 * G * Cs, s1 * G * Cs
            cut[k] = a[..., lo:hi]
        r = self.like(cut)
        r.n_segments = s1 - s0
        return r


def alloc_outputs(soa: SweepSoA, with_pairs: bool = True) -> dict:
    out = {}
    for k in SWEEP_OUT_FIELDS:
        if k.startswith("pair") and not with_pairs:
            continue
        n = soa.n_pairs if k.startswith("pair") else soa.n_segments
        out[k] = D.empty(n, OUT_DTYPES[k])
    return out


def sweep_args(soa: SweepSoA, params: torch.Tensor, outputs: dict, effect_cap: float = 50.0,
               use_violate: bool = True, use_meet: bool = True) -> SweepArgs:
    a = SweepArgs()
    a.n_metrics, a.n_slots, a.gpus_per_segment = soa.n_metrics, soa.n_slots, soa.gpus_per_segment
    a.concurrency_limit, a.n_segments, a.now = soa.concurrency_limit, soa.n_segments, float(soa.now)
    a.effect_cap, a.use_violate, a.use_meet = float(effect_cap), int(use_violate), int(use_meet)
    a.params = D.ptr(params)
    for k in INPUT_FIELDS:
        setattr(a, k, D.ptr(soa.arrays[k]))
    for k in SWEEP_OUT_FIELDS:
        setattr(a, k, D.ptr(outputs.get(k)))
    return a


def launch_sweep(soa: SweepSoA, params: torch.Tensor, outputs: dict, effect_cap: float = 50.0,
                 use_violate: bool = True, use_meet: bool = True, stream=None) -> None:
    """Asynchronous strait_sweep on device-resident ``soa``."""
    args = sweep_args(soa, params, outputs, effect_cap, use_violate, use_meet)
    D.check(D.lib().strait_sweep(C.byref(args), D.stream_handle(stream)))


def launch_round(soa: SweepSoA, params: torch.Tensor, outputs: dict, refit: RefitArgs, effect_cap: float = 50.0,
                 stream=None) -> None:
    """Asynchronous strait_round: sweep under ``params`` fused with the refit."""
    args = sweep_args(soa, params, outputs, effect_cap)
    D.check(D.lib().strait_round(C.byref(args), C.byref(refit), D.stream_handle(stream)))


def sweep(soa: SweepSoA, params, effect_cap: float = 50.0, use_violate: bool = True, use_meet: bool = True,
          with_pairs: bool = True) -> dict:
    """Host-in/host-out sweep (H2D, one kernel, D2H) -> numpy outputs."""
    dsoa = soa if isinstance(next(iter(soa.arrays.values())), torch.Tensor) else soa.to_device()
    P = params if isinstance(params, torch.Tensor) else D.dev(np.asarray(params, dtype=np.float64))
    out = alloc_outputs(dsoa, with_pairs)
    launch_sweep(dsoa, P, out, effect_cap, use_violate, use_meet)
    return {k: D.host(v) for k, v in out.items()}


def expand_args(tables: dict, ent_row: torch.Tensor, cand_row: torch.Tensor, stride: int):
    from ._abi import SweepExpandArgs

    e = SweepExpandArgs()
    e.table_stride, e.n_rows = int(stride), int(tables["self_cmp"].numel())
    for k in ("thr", "self_cmp", "self_mem", "kernel", "total", "deadline", "prio"):
        setattr(e, k, D.ptr(tables[k]))
    e.ent_row, e.cand_row = D.ptr(ent_row), D.ptr(cand_row)
    return e


def load_compact(dsoa: SweepSoA, fields: dict, rows: dict, dev_rows: dict, dev_tables: dict, stride: int,
                 stream=None) -> None:
    """Fill a device-resident (packed) snapshot from a profile-indexed one
    (microbench.c3_compact): the non-derived `fields` are copied (H2D from
    pinned host tensors) straight into their rows of the packed blocks, the
    int16 profile `rows` into `dev_rows`, and strait_sweep_expand rebuilds
    every profile-derived field and the list-order aggregates on the device."""
    for k, v in fields.items():
        dsoa.arrays[k].copy_(v, non_blocking=True)
    for k in ("ent_row", "cand_row"):
        dev_rows[k].copy_(rows[k], non_blocking=True)
    e = expand_args(dev_tables, dev_rows["ent_row"], dev_rows["cand_row"], stride)
    a = sweep_args(dsoa, dev_rows["ent_row"], {})  # params unused by the expand
    D.check(D.lib().strait_sweep_expand(C.byref(e), C.byref(a), D.stream_handle(stream)))


def last_sweep_path() -> str:
    return {1: "sync", 2: "tma-bulk", 3: "tma-tensor"}.get(D.lib().strait_last_sweep_path(), "none")
