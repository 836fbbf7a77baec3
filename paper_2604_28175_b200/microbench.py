"""Synthetic inputs of the candidate-sweep microbench (BASELINE config 3,
SURVEY.md §8(d)): 2^24 (candidate, GPU, co-runner) triples per scheduling
round = 2^22 (candidate, GPU) pairs x 4 co-runner slots, grouped into 2^16
segments (one candidate batch scored against 64 independent GPU states), and
F = 64 feedback samples refit sequentially every round.

The SoA is generated directly (numpy, seeded ``SeedSequence([2604, round])``)
but is object-consistent: every pair is a valid GpuRuntimeState snapshot whose
aggregates are the reference's list-order sums of its running entries'
profiled contributions (runtime.py:104-122), so any segment can be rebuilt as
reference objects and re-evaluated by the reference (tests/golden).
"""
from __future__ import annotations

import math

import numpy as np

from .domain import DEFAULT_METRICS, PriorityLevel
from .profiles import random_profile
from .sweep import SweepSoA

N_MODELS = 32
N_HP = 8
NOW = 100.0
C3_SEGMENTS = 1 << 16
C3_GPUS = 64
C3_SLOTS = 4
C3_CONCURRENCY = 5  # every snapshot admits the candidate: all live co-runners get projected
C3_FEEDBACK = 64

# hidden matched-family truth used for the feedback stream (test_acceptance.py:280-297)
HIDDEN = dict(scale=0.35, base=2.3, offset=-0.15, weights=(0.22, 0.28, 0.18, 0.25, 0.2),
              w_cmp=0.3, w_mem=0.15, coeff=(0.6, 1.0))


def c3_profiles():
    rng = np.random.default_rng(2604)
    return [random_profile(rng, f"m{i:02d}", PriorityLevel.HIGH if i < N_HP else PriorityLevel.LOW)
            for i in range(N_MODELS)]


def profile_tables(profiles):
    """(model, size) lookup tables: [M, 8] scalars and [M, 8, nm] throughput."""
    M = len(profiles)
    bs = profiles[0].max_batch_size
    t = {k: np.empty((M, bs)) for k in ("total", "kernel", "cmp", "mem")}
    thr = np.empty((M, bs, len(DEFAULT_METRICS)))
    for i, p in enumerate(profiles):
        t["total"][i] = p.total_latency
        t["kernel"][i] = p.kernel_latency
        t["cmp"][i] = p.self_compute
        t["mem"][i] = p.self_memory
        thr[i] = np.asarray(p.throughput)
    t["thr"] = thr
    t["deadline"] = np.array([p.deadline_ms for p in profiles])
    t["prio"] = np.array([int(p.priority) for p in profiles], dtype=np.int8)
    return t


def c3_round(round_idx: int, n_segments: int = C3_SEGMENTS, gpus: int = C3_GPUS, slots: int = C3_SLOTS,
             profiles=None, concurrency_limit: int = C3_CONCURRENCY) -> SweepSoA:
    profiles = profiles if profiles is not None else c3_profiles()
    tab = profile_tables(profiles)
    nm = len(DEFAULT_METRICS)
    rng = np.random.default_rng(np.random.SeedSequence([2604, round_idx]))
    S, P = n_segments, n_segments * gpus
    T = P * slots
    M = len(profiles)

    # candidates: (model, size, front enqueue)
    cm = rng.integers(0, M, S)
    ck = rng.integers(1, 9, S) - 1
    front = NOW - rng.uniform(0.0, 2.0, S)
    # GPU states
    cap = rng.uniform(75.0, 100.0, P)
    t_avail = NOW + rng.uniform(0.0, 1.0, P)
    nrun = rng.binomial(slots, 0.9, P).astype(np.int8)
    # co-runners
    em = rng.integers(0, M, T)
    ek = rng.integers(1, 9, T) - 1
    kstart = rng.uniform(97.0, 100.0, T)
    deadline_abs = NOW + rng.uniform(0.0, 20.0, T)
    twa = rng.uniform(0.0, 1.5, (nm, T))

    ent_contrib = np.ascontiguousarray(tab["thr"][em, ek].T)  # [nm, T]
    eprio = tab["prio"][em]
    live = (np.arange(T) % slots) < np.repeat(nrun.astype(np.int64), slots)
    # list-order aggregates from 0.0 (runtime.py:104-109, 116-122)
    c4 = ent_contrib.reshape(nm, P, slots)
    l4 = live.reshape(P, slots)
    lp4 = l4 & (eprio.reshape(P, slots) == 1)
    agg = np.zeros((nm, P))
    lp = np.zeros((nm, P))
    for c in range(slots):
        agg = agg + np.where(l4[:, c], c4[:, :, c], 0.0)
        lp = lp + np.where(lp4[:, c], c4[:, :, c], 0.0)

    arrays = {
        "cand_contrib": np.ascontiguousarray(tab["thr"][cm, ck].T),
        "cand_self_cmp": tab["cmp"][cm, ck],
        "cand_self_mem": tab["mem"][cm, ck],
        "cand_total": tab["total"][cm, ck],
        "cand_kernel": tab["kernel"][cm, ck],
        "cand_deadline": tab["deadline"][cm],
        "cand_front": front,
        "cand_prio": tab["prio"][cm],
        "gpu_agg": agg,
        "gpu_lp_agg": lp,
        "gpu_cap_pct": cap,
        "gpu_t_avail": t_avail,
        "gpu_n_running": nrun,
        "ent_contrib": ent_contrib,
        "ent_twa": twa,
        "ent_self_cmp": tab["cmp"][em, ek],
        "ent_self_mem": tab["mem"][em, ek],
        "ent_t_kernel": tab["kernel"][em, ek],
        "ent_deadline_abs": deadline_abs,
        "ent_kstart": kstart,
        "ent_prio": eprio,
    }
    arrays = {k: np.ascontiguousarray(v) for k, v in arrays.items()}
    meta = dict(cand_model=cm, cand_size=ck + 1, ent_model=em, ent_size=ek + 1)
    soa = SweepSoA(nm, slots, gpus, concurrency_limit, S, NOW, arrays)
    soa.meta = meta  # object-level provenance for reference rebuilds
    return soa


# fields a profile-indexed snapshot ships (the rest follow from the profile rows)
COMPACT_FIELDS = ("ent_twa", "ent_deadline_abs", "ent_kstart", "gpu_cap_pct", "gpu_t_avail", "gpu_n_running",
                  "cand_front")


def c3_compact(soa: SweepSoA, profiles=None) -> dict:
    """Profile-indexed form of a C3 round (strait_sweep_expand): int16 profile
    rows per co-runner and candidate + the non-derived fields, and the profile
    tables (row = model * max_batch + size - 1)."""
    profiles = profiles if profiles is not None else c3_profiles()
    tab = profile_tables(profiles)
    bs = tab["total"].shape[1]
    m = soa.meta
    out = {k: soa.arrays[k] for k in COMPACT_FIELDS}
    out["ent_row"] = (m["ent_model"] * bs + m["ent_size"] - 1).astype(np.int16)
    out["cand_row"] = (m["cand_model"] * bs + m["cand_size"] - 1).astype(np.int16)
    tables = {"thr": np.ascontiguousarray(tab["thr"].reshape(-1, tab["thr"].shape[2]).T),
              "self_cmp": tab["cmp"].ravel(), "self_mem": tab["mem"].ravel(), "kernel": tab["kernel"].ravel(),
              "total": tab["total"].ravel(), "deadline": tab["deadline"], "prio": tab["prio"]}
    return {"fields": {k: np.ascontiguousarray(v) for k, v in out.items()},
            "tables": {k: np.ascontiguousarray(v) for k, v in tables.items()}, "table_stride": bs}


def c3_feedback(round_idx: int, n: int = C3_FEEDBACK):
    """F feedback samples per round, as the reference's convergence stream
    (test_acceptance.py:280-297): matched-family hidden truth with
    lognormal noise sigma 0.05.  Synthetic input data (host numpy)."""
    rng = np.random.default_rng(np.random.SeedSequence([2604, round_idx, 1]))
    nm = len(DEFAULT_METRICS)
    agg = rng.uniform(0.0, 2.0, (n, nm))
    cmp_ = rng.uniform(0.1, 0.9, n)
    mem = rng.uniform(0.1, 0.9, n)
    prio = np.where(rng.uniform(size=n) < 0.4, 0, 1).astype(np.int8)
    noise = rng.normal(0.0, 0.05, n)
    h = HIDDEN
    actual = np.empty(n)
    for i in range(n):
        x = h["w_cmp"] * cmp_[i] + h["w_mem"] * mem[i]
        for w, a in zip(h["weights"], agg[i]):
            x += w * a
        eff = min(max(h["scale"] * h["base"] ** x + h["offset"], 0.0), 50.0)
        truth = 1.0 + eff * h["coeff"][prio[i]]
        actual[i] = 1.0 + (truth - 1.0) * math.exp(noise[i])
    return {"twa": np.ascontiguousarray(agg.T), "self_cmp": cmp_, "self_mem": mem, "prio": prio, "actual": actual}


def algorithmic_bytes(soa: SweepSoA, with_pairs: bool = True) -> int:
    """Bytes one sweep must move: every input field once + the outputs."""
    out_pair = (1 + 8 + 8) * soa.n_pairs if with_pairs else 0
    out_seg = (4 + 8 + 8) * soa.n_segments
    return soa.input_bytes() + out_pair + out_seg
