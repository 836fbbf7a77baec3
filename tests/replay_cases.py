"""Replay configurations of the golden fixtures (tests/golden/replay/*.npz),
rebuilt with this package only so they are available on the GPU box.
tests/golden/gen_golden.py builds the same configurations with the
reference's own loaders (the shipped pkg/configs YAMLs, restated here as
dicts; the example trace's per-minute counts likewise)."""
from __future__ import annotations

import math

import numpy as np

from paper_2604_28175_b200 import config as MC
from paper_2604_28175_b200.domain import PriorityLevel
from paper_2604_28175_b200.profiles import random_profile
from paper_2604_28175_b200.workload import ModelWorkload

# pkg/configs/example_trace.csv (per-minute counts)
EXAMPLE_TRACE = {"vision_gate": {0: 7654.0, 1: 11412.0, 2: 7322.0, 3: 7268.0, 4: 8189.0},
                 "doc_reader": {0: 2514.0, 1: 3306.0, 2: 2307.0, 3: 3713.0, 4: 3644.0}}

DEMO = {"profiles": "default6", "duration_ms": 1000, "seed": 1, "n_gpus": 1, "policy": "predictive",
        "ground_truth": {"noise_sigma": 0.05},
        "workload": {"resnet50": {"mode": "poisson", "rate": 300}, "yolo_v8n": {"mode": "uniform", "rate": 150},
                     "roberta_b": {"mode": "poisson", "rate": 80}}}
C1 = {"profiles": "default6", "duration_ms": 26316, "seed": 1, "n_gpus": 1, "policy": "predictive",
      "ground_truth": {"noise_sigma": 0.05},
      "workload": {"resnet50": {"mode": "poisson", "rate": 300}, "roberta_b": {"mode": "poisson", "rate": 80}}}
OVERLOAD_GT = {"family": "exponential", "scale": 0.5, "base": 2.718281828459045, "offset": -0.7686,
               "weights": [0.3] * 5, "self_compute_weight": 0.25, "self_memory_weight": 0.2,
               "priority_factor": {"high": 0.6, "low": 1.0}, "noise_sigma": 0.05}
OVERLOAD_WL = {"resnet50": {"mode": "poisson", "rate": 2200}, "vit_b16": {"mode": "poisson", "rate": 800},
               "yolo_v8n": {"mode": "poisson", "rate": 1300}, "convnext_b": {"mode": "poisson", "rate": 650},
               "vgg19": {"mode": "poisson", "rate": 650}, "roberta_b": {"mode": "poisson", "rate": 400}}


def overload_doc(duration=3000, **kw):
    d = {"profiles": "default6", "duration_ms": duration, "seed": 0, "n_gpus": 4, "concurrency_limit": 4,
         "policy": "predictive", "goodput_window_ms": 1000, "ground_truth": dict(OVERLOAD_GT),
         "workload": dict(OVERLOAD_WL)}
    d.update(kw)
    return d


def trace_config(duration=30000):
    doc = {"profiles": "default6", "duration_ms": duration, "seed": 2, "n_gpus": 2, "policy": "predictive",
           "ground_truth": {"noise_sigma": 0.05}, "workload": {"yolo_v8n": {"mode": "poisson", "rate": 100}}}
    cfg = MC.config_from_dict(doc)
    cfg.workload.models["resnet50"] = ModelWorkload("trace", function_id="vision_gate", scale=1.0,
                                                    trace_table=EXAMPLE_TRACE)
    cfg.workload.models["roberta_b"] = ModelWorkload("trace", function_id="doc_reader", scale=0.5,
                                                     trace_table=EXAMPLE_TRACE)
    cfg.validate()
    return cfg


def c5_config(duration=150.0, minutes=2, seed=0, n_gpus=64):
    """C5 shape: 20 random_profile models (m00-m05 HP bursty
    trace, m06-m19 LP Poisson 2600/s), 64 GPUs."""
    rng = np.random.default_rng(2604)
    profs = {f"m{i:02d}": random_profile(rng, f"m{i:02d}", PriorityLevel.HIGH if i < 6 else PriorityLevel.LOW)
             for i in range(20)}
    table = {}
    for i in range(6):
        for m in range(minutes):
            table.setdefault(f"hp{i}", {})[m] = float(int(rng.lognormal(math.log(150000), 0.6)))
    wl = {f"m{i:02d}": ({"mode": "poisson", "rate": 2600}) for i in range(6, 20)}
    doc = {"profiles": profs, "duration_ms": duration, "seed": seed, "n_gpus": n_gpus, "concurrency_limit": 4,
           "policy": "predictive", "ground_truth": {"noise_sigma": 0.05}, "workload": wl}
    cfg = MC.config_from_dict(doc)
    for i in range(6):
        cfg.workload.models[f"m{i:02d}"] = ModelWorkload("trace", function_id=f"hp{i}", scale=1.0, trace_table=table)
    cfg.validate()
    return cfg


def case_config(name: str):
    if name == "demo":
        return MC.config_from_dict(DEMO)
    if name == "c1":
        return MC.config_from_dict(C1)
    if name == "overload":
        return MC.config_from_dict(overload_doc())
    if name == "trace":
        return trace_config()
    if name == "c5_slice":
        return c5_config()
    variants = {"ov_no_meet": dict(policy_variant="no_meet"), "ov_no_violate": dict(policy_variant="no_violate_aimd"),
                "ov_no_prio": dict(policy_variant="no_priority_scan"),
                "ov_no_gamma": dict(policy_variant="no_gamma_advantage"),
                "ov_quadratic": dict(ground_truth=dict(OVERLOAD_GT, family="quadratic", scale=0.3, offset=-0.4))}
    if name in variants:
        return MC.config_from_dict(overload_doc(500, **variants[name]))
    if name == "ov_nonoise_2gpu":
        return MC.config_from_dict(overload_doc(400, n_gpus=2, ground_truth=dict(OVERLOAD_GT, noise_sigma=0.0)))
    raise KeyError(name)


CASES = ["demo", "c1", "overload", "trace", "ov_no_meet", "ov_no_violate", "ov_no_prio", "ov_no_gamma",
         "ov_quadratic", "ov_nonoise_2gpu", "c5_slice"]

# arrays compared bit-exactly between the reference, the C oracle and (decisions) the device
REQ_KEYS = ("req_status", "req_violated", "req_batch")
DEC_KEYS = ("dec_pass", "dec_model", "dec_size", "dec_gpu")
FLOAT_KEYS = ("req_completion", "dec_time", "dec_est_latency", "dec_intf", "b_front", "b_transfer_start",
              "b_kernel_start", "b_kernel_end", "b_completion", "fb_predicted", "fb_actual",
              "fb_residual", "cap_time", "cap_pct")
# b_work (sum of segment d/s) is checked to 1e-12: the reference sums with Python 3.12's
# compensated float sum(), the engines accumulate left to right.
