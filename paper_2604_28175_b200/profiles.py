"""Profile inputs: the builtin ``default6`` set, ``random_profile`` and YAML
profile documents (reference: /root/reference/pkg/src/infersim/profiles.py).

Input-data plumbing for the device path; the generators consume a numpy
Generator in the reference's draw order so the same seed yields the same
profiles (pinned by tests/test_inputs.py against reference golden vectors).
"""
from __future__ import annotations

import os
from typing import Optional

import numpy as np
import yaml

from .domain import (
    DEFAULT_METRICS,
    ModelProfile,
    PriorityLevel,
    ProfileParseError,
    ProfileValidationError,
    validate_profile,
)

_TOP_FIELDS = {"model_id", "priority", "deadline_ms", "batch_timeout_ms", "max_batch_size", "metrics", "sizes"}
_SIZE_FIELDS = {"batch_size", "total_latency_ms", "transfer_latency_ms", "kernel_latency_ms", "throughput",
                "self_compute", "self_memory"}


def _synthetic_profile(model_id, priority, deadline_ms, base_latency_ms, transfer_frac, kernel_frac, peaks,
                       half_size, max_batch_size=8, timeout_frac=0.1) -> ModelProfile:
    """profiles.py:178-215: latencies base*(0.5+0.5j), saturating throughputs,
    every value rounded to 6 decimals with Python's round()."""
    total, transfer, kernel, throughput, self_cmp, self_mem = [], [], [], [], [], []
    for j in range(1, max_batch_size + 1):
        t = base_latency_ms * (0.5 + 0.5 * j)
        total.append(round(t, 6))
        transfer.append(round(transfer_frac * t, 6))
        kernel.append(round(kernel_frac * t, 6))
        row = tuple(round(peaks[m] * j / (j + half_size), 6) for m in DEFAULT_METRICS)
        throughput.append(row)
        self_cmp.append(row[DEFAULT_METRICS.index("tensor_pipe")])
        self_mem.append(row[DEFAULT_METRICS.index("l2_cache")])
    return ModelProfile(model_id, priority, deadline_ms, round(timeout_frac * deadline_ms, 6), max_batch_size,
                        total, transfer, kernel, throughput, self_cmp, self_mem)


def default_profiles() -> dict[str, ModelProfile]:
    """profiles.py:218-240 — two high-priority vision models + four best-effort."""
    hi, lo = PriorityLevel.HIGH, PriorityLevel.LOW
    specs = [
        ("resnet50", hi, 8.0, 2.0, 0.16, 0.72,
         dict(l1_cache=0.55, l2_cache=0.45, dram=0.40, tensor_pipe=0.35, fma_pipe=0.70), 2.0),
        ("vit_b16", hi, 15.0, 3.6, 0.10, 0.76,
         dict(l1_cache=0.40, l2_cache=0.55, dram=0.45, tensor_pipe=0.75, fma_pipe=0.35), 2.5),
        ("yolo_v8n", lo, 20.0, 1.6, 0.14, 0.70,
         dict(l1_cache=0.45, l2_cache=0.35, dram=0.30, tensor_pipe=0.30, fma_pipe=0.55), 1.5),
        ("convnext_b", lo, 25.0, 4.4, 0.10, 0.78,
         dict(l1_cache=0.50, l2_cache=0.50, dram=0.50, tensor_pipe=0.60, fma_pipe=0.55), 3.0),
        ("vgg19", lo, 25.0, 4.0, 0.12, 0.76,
         dict(l1_cache=0.60, l2_cache=0.55, dram=0.60, tensor_pipe=0.40, fma_pipe=0.75), 3.0),
        ("roberta_b", lo, 45.0, 5.2, 0.06, 0.80,
         dict(l1_cache=0.35, l2_cache=0.70, dram=0.65, tensor_pipe=0.70, fma_pipe=0.30), 3.5),
    ]
    return {s[0]: _synthetic_profile(*s) for s in specs}


def random_profile(rng: np.random.Generator, model_id: str, priority: Optional[PriorityLevel] = None,
                   max_batch_size: int = 8) -> ModelProfile:
    """profiles.py:243-261 — same draw order as the reference."""
    if priority is None:
        priority = PriorityLevel(int(rng.integers(0, 2)))
    base = float(rng.uniform(0.8, 6.0))
    transfer_frac = float(rng.uniform(0.05, 0.2))
    kernel_frac = float(rng.uniform(0.6, 0.78))
    peaks = {m: float(rng.uniform(0.15, 0.9)) for m in DEFAULT_METRICS}
    half = float(rng.uniform(1.0, 4.0))
    deadline = base * (1.5 + float(rng.uniform(0.5, 6.0)))
    return _synthetic_profile(model_id, priority, deadline, base, transfer_frac, kernel_frac, peaks, half,
                              max_batch_size=max_batch_size)


def profile_to_dict(profile: ModelProfile) -> dict:
    sizes = []
    for j in range(1, profile.max_batch_size + 1):
        sizes.append({
            "batch_size": j,
            "total_latency_ms": profile.total_latency_ms(j),
            "transfer_latency_ms": profile.transfer_latency_ms(j),
            "kernel_latency_ms": profile.kernel_latency_ms(j),
            "throughput": {m: v for m, v in zip(profile.metrics, profile.throughput_at(j))},
            "self_compute": profile.self_compute_at(j),
            "self_memory": profile.self_memory_at(j),
        })
    return {"model_id": profile.model_id, "priority": profile.priority.label, "deadline_ms": profile.deadline_ms,
            "batch_timeout_ms": profile.batch_timeout_ms, "max_batch_size": profile.max_batch_size,
            "metrics": list(profile.metrics), "sizes": sizes}


def profile_from_dict(doc: dict, source: str = "<dict>") -> ModelProfile:
    """profiles.py:74-136 — strict field checking."""
    if not isinstance(doc, dict):
        raise ProfileParseError(f"{source}: profile document must be a mapping")
    unknown = set(doc) - _TOP_FIELDS
    if unknown:
        raise ProfileParseError(f"{source}: unknown fields {sorted(unknown)}")
    missing = _TOP_FIELDS - {"metrics"} - set(doc)
    if missing:
        raise ProfileParseError(f"{source}: missing fields {sorted(missing)}")
    metrics = tuple(doc.get("metrics", DEFAULT_METRICS))
    sizes = doc["sizes"]
    if not isinstance(sizes, list) or not sizes:
        raise ProfileParseError(f"{source}: 'sizes' must be a non-empty list")
    max_bs = int(doc["max_batch_size"])
    total, transfer, kernel, throughput, self_cmp, self_mem = [], [], [], [], [], []
    for expected, item in enumerate(sizes, start=1):
        if not isinstance(item, dict):
            raise ProfileParseError(f"{source}: size entries must be mappings")
        if set(item) - _SIZE_FIELDS:
            raise ProfileParseError(f"{source}: unknown size fields {sorted(set(item) - _SIZE_FIELDS)}")
        if _SIZE_FIELDS - set(item):
            raise ProfileParseError(f"{source}: size entry missing {sorted(_SIZE_FIELDS - set(item))}")
        if int(item["batch_size"]) != expected:
            raise ProfileParseError(f"{source}: size entries must cover 1..{max_bs} in order; "
                                    f"expected {expected}, got {item['batch_size']}")
        total.append(float(item["total_latency_ms"]))
        transfer.append(float(item["transfer_latency_ms"]))
        kernel.append(float(item["kernel_latency_ms"]))
        tp = item["throughput"]
        if not isinstance(tp, dict) or set(tp) != set(metrics):
            raise ProfileParseError(f"{source}: throughput must map exactly the metrics {list(metrics)}")
        throughput.append(tuple(float(tp[m]) for m in metrics))
        self_cmp.append(float(item["self_compute"]))
        self_mem.append(float(item["self_memory"]))
    if len(sizes) != max_bs:
        raise ProfileParseError(f"{source}: {len(sizes)} size entries but max_batch_size={max_bs}")
    return ModelProfile(str(doc["model_id"]), PriorityLevel.from_name(str(doc["priority"])),
                        float(doc["deadline_ms"]), float(doc["batch_timeout_ms"]), max_bs, total, transfer,
                        kernel, throughput, self_cmp, self_mem, metrics)


def load_profile(path) -> ModelProfile:
    try:
        with open(path) as f:
            doc = yaml.safe_load(f)
    except yaml.YAMLError as e:
        raise ProfileParseError(f"{path}: {e}") from e
    profile = profile_from_dict(doc, source=str(path))
    violations = validate_profile(profile)
    if violations:
        raise ProfileValidationError(profile.model_id, violations)
    return profile


def save_profile(profile: ModelProfile, path) -> None:
    with open(path, "w") as f:
        yaml.safe_dump(profile_to_dict(profile), f, sort_keys=False)


def load_profiles_dir(directory) -> dict[str, ModelProfile]:
    names = sorted(n for n in os.listdir(directory) if n.endswith((".yaml", ".yml")))
    if not names:
        raise ProfileParseError(f"{directory}: no profile documents found")
    profiles: dict[str, ModelProfile] = {}
    for name in names:
        p = load_profile(os.path.join(directory, name))
        if p.model_id in profiles:
            raise ProfileParseError(f"{directory}: duplicate model_id {p.model_id!r}")
        profiles[p.model_id] = p
    return profiles


def save_profiles_dir(profiles: dict[str, ModelProfile], directory) -> None:
    os.makedirs(directory, exist_ok=True)
    for model_id in sorted(profiles):
        save_profile(profiles[model_id], os.path.join(directory, f"{model_id}.yaml"))
