"""Replay configurations of the golden fixtures (tests/golden/replay/*.npz),
rebuilt with this package only so they are available on the GPU box.
tests/golden/gen_golden.py builds the same configurations with the
reference's own loaders (the shipped pkg/configs YAMLs, restated here as
dicts; the example trace's per-minute counts likewise)."""
from __future__ import annotations

from paper_2604_28175_b200 import config as MC
from paper_2604_28175_b200.configs import (C1, DEMO, EXAMPLE_TRACE, OVERLOAD_GT, OVERLOAD_WL,  # noqa: F401
                                           overload_doc)
from paper_2604_28175_b200.configs import c5 as c5_config
from paper_2604_28175_b200.configs import trace_replay as trace_config


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
    if name in ("ov_temporal", "ov_static"):
        return MC.config_from_dict(overload_doc(500, policy=name[3:]))
    if name == "ov_reactive":
        return MC.config_from_dict(overload_doc(1500, policy="reactive"))
    if name == "c1_reactive":
        return MC.config_from_dict(dict(C1, duration_ms=5000, policy="reactive"))
    if name == "ov_nonoise_2gpu":
        return MC.config_from_dict(overload_doc(400, n_gpus=2, ground_truth=dict(OVERLOAD_GT, noise_sigma=0.0)))
    raise KeyError(name)


CASES = ["demo", "c1", "overload", "trace", "ov_no_meet", "ov_no_violate", "ov_no_prio", "ov_no_gamma",
         "ov_quadratic", "ov_nonoise_2gpu", "c5_slice", "ov_temporal", "ov_static", "ov_reactive", "c1_reactive"]

# arrays compared bit-exactly between the reference, the C oracle and (decisions) the device
REQ_KEYS = ("req_status", "req_violated", "req_batch")
DEC_KEYS = ("dec_pass", "dec_model", "dec_size", "dec_gpu")
FLOAT_KEYS = ("req_completion", "dec_time", "dec_est_latency", "dec_intf", "b_front", "b_transfer_start",
              "b_kernel_start", "b_kernel_end", "b_completion", "fb_predicted", "fb_actual",
              "fb_residual", "cap_time", "cap_pct")
# b_work (sum of segment d/s) is checked to 1e-12: the reference sums with Python 3.12's
# compensated float sum(), the engines accumulate left to right.
