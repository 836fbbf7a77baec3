"""Random object-API scheduling states, built the same way on the reference's
classes (tests/golden/gen_node_golden.py) and on this package's
(tests/test_node_*.py): GPUs with link reservations, AIMD caps and running
entries whose timelines hold arbitrary sample histories, plus a candidate
queue.  A scenario is plain JSON (floats as float.hex) so the reference's
answers can travel to the GPU box as a fixture."""
from __future__ import annotations

import numpy as np

NOW = 100.0


def hx(v: float) -> str:
    return float(v).hex()


def fx(s: str) -> float:
    return float.fromhex(s)


def random_scenario(rng: np.random.Generator, n_gpus: int, nm: int = 5, error: str | None = None) -> dict:
    M = 6
    profiles = []
    for i in range(M):
        bs = 8
        base = float(rng.uniform(1.0, 6.0))
        tot = sorted(float(base * (0.6 + 0.4 * j) + rng.uniform(0, 0.2)) for j in range(1, bs + 1))
        profiles.append({
            "model_id": f"m{i}", "priority": int(i >= 2), "deadline_ms": hx(tot[0] * float(rng.uniform(2.0, 6.0))),
            "batch_timeout_ms": hx(float(rng.uniform(0.5, 3.0))), "max_batch_size": bs,
            "total": [hx(t) for t in tot], "transfer": [hx(0.15 * t) for t in tot], "kernel": [hx(0.6 * t) for t in tot],
            "throughput": [[hx(v) for v in rng.uniform(0.0, 0.6, nm)] for _ in range(bs)],
            "self_compute": [hx(v) for v in rng.uniform(0, 1, bs)], "self_memory": [hx(v) for v in rng.uniform(0, 1, bs)],
        })
    gpus = []
    for g in range(n_gpus):
        limit = int(rng.integers(2, 5))
        n_run = int(rng.integers(0, limit + 1))
        res = []
        t = NOW - float(rng.uniform(0, 4))
        for _ in range(int(rng.integers(0, 4))):
            res.append([hx(t), hx(float(rng.uniform(0.1, 2.0)))])
            t += float(rng.uniform(0, 1.5))
        ents = []
        for _ in range(n_run):
            m = int(rng.integers(0, M))
            k = int(rng.integers(1, 9))
            started = bool(rng.uniform() < 0.6)
            times = sorted(float(x) for x in rng.uniform(NOW - 6, NOW, int(rng.integers(1, 5))))
            if rng.uniform() < 0.2:
                times[-1] = NOW  # a sample exactly at now
            samples = [[hx(tt), [hx(v) for v in rng.uniform(0.0, 1.4, nm)]] for tt in times]
            ents.append({"model": m, "size": k, "started": started, "kernel_start": hx(NOW - float(rng.uniform(0, 5))),
                         "kstart_est": hx(NOW + float(rng.uniform(-1, 2))),
                         "deadline_abs": hx(NOW + float(rng.uniform(-2, 25))), "intf": hx(float(rng.uniform(1, 2))),
                         "samples": samples})
        gpus.append({"gpu_id": g, "limit": limit, "cap_pct": hx(float(rng.uniform(75, 100))),
                     "reservations": res, "calibrate": bool(res) and bool(rng.uniform() < 0.3), "entries": ents})
    if error == "empty_timeline":
        for gg in gpus:
            if gg["entries"]:
                gg["entries"][0]["samples"] = []
                break
    elif error == "future_sample":
        for gg in gpus:
            if gg["entries"]:
                gg["entries"][-1]["samples"][-1][0] = hx(NOW + 1.0)
                break
    cand = int(rng.integers(0, M))
    flags = [(True, True), (True, False), (False, True)][int(rng.integers(0, 3))]
    if error:  # a LOW candidate under check_violate reads every running entry's timeline
        cand, flags = 2 + int(rng.integers(0, M - 2)), (True, True)
        for gg in gpus:
            gg["cap_pct"] = hx(100.0)
    params = {"scale": hx(float(rng.uniform(0.05, 1.5))), "base": hx(float(rng.uniform(1.2, 3.5))),
              "offset": hx(float(rng.uniform(-0.8, 0.5))), "weights": [hx(v) for v in rng.uniform(-0.3, 0.8, nm)],
              "w_cmp": hx(float(rng.uniform(-0.3, 0.8))), "w_mem": hx(float(rng.uniform(-0.3, 0.8))),
              "coeff": [hx(float(rng.uniform(0.1, 1.0))), hx(float(rng.uniform(0.5, 2.0)))]}
    return {"nm": nm, "now": hx(NOW), "profiles": profiles, "gpus": gpus, "cand": cand,
            "k_queue": int(rng.integers(1, 11)), "front": hx(NOW - float(rng.uniform(0, 3))), "params": params,
            "use_violate": flags[0], "use_meet": flags[1], "error": error}


def build(scn: dict, api) -> dict:
    """Objects of `scn` on the classes of `api` (a module namespace with the
    reference's names)."""
    P = api.PriorityLevel
    nm = scn["nm"]
    now = fx(scn["now"])
    metrics = tuple(f"x{i}" for i in range(nm))
    profiles = []
    for p in scn["profiles"]:
        profiles.append(api.ModelProfile(
            p["model_id"], P(p["priority"]), fx(p["deadline_ms"]), fx(p["batch_timeout_ms"]), p["max_batch_size"],
            [fx(v) for v in p["total"]], [fx(v) for v in p["transfer"]], [fx(v) for v in p["kernel"]],
            [tuple(fx(v) for v in row) for row in p["throughput"]], [fx(v) for v in p["self_compute"]],
            [fx(v) for v in p["self_memory"]], metrics))
    gpus, n = [], 0
    for gs in scn["gpus"]:
        gpu = api.GpuRuntimeState(gs["gpu_id"], nm, gs["limit"])
        gpu.aimd.cap_pct = fx(gs["cap_pct"])
        for t, d in gs["reservations"]:
            gpu.pcie.reserve(fx(t), fx(d))
        if gs["calibrate"]:
            gpu.pcie.calibrate(gpu.pcie.pending[0] + 0.25)
        for e in gs["entries"]:
            prof = profiles[e["model"]]
            k = e["size"]
            n += 1
            reqs = [api.Request(f"r{n}-{j}", prof.model_id, now - 3.0, now - 3.0 + prof.deadline_ms) for j in range(k)]
            b = api.Batch(f"b{n}", prof.model_id, k, prof.priority, now - 3.0, reqs, gpu_id=gs["gpu_id"])
            if e["started"]:
                b.kernel_start = fx(e["kernel_start"])
            ent = api.RunningTaskEntry(b, prof.throughput_at(k), prof.self_compute_at(k), prof.self_memory_at(k),
                                       prof.kernel_latency_ms(k), fx(e["deadline_abs"]), fx(e["intf"]),
                                       fx(e["kstart_est"]), api.ThroughputTimeline(), e["started"])
            gpu.add_entry(ent, now - 6.5)
        # then the arbitrary timeline histories (a later add would restamp them at now - 6.5)
        for ent, e in zip(list(gpu.running), gs["entries"]):
            ent.timeline = api.ThroughputTimeline([(fx(t), tuple(fx(v) for v in vec)) for t, vec in e["samples"]])
        gpus.append(gpu)
    cprof = profiles[scn["cand"]]
    q = api.TaskQueue(cprof)
    front = fx(scn["front"])
    for j in range(scn["k_queue"]):
        q.push(api.Request(f"q{j}", cprof.model_id, front + 0.01 * j, front + 0.01 * j + cprof.deadline_ms))
    pp = scn["params"]
    params = api.PredictorParams(scale=fx(pp["scale"]), base=fx(pp["base"]), offset=fx(pp["offset"]),
                                 weights=tuple(fx(v) for v in pp["weights"]), self_compute_weight=fx(pp["w_cmp"]),
                                 self_memory_weight=fx(pp["w_mem"]),
                                 priority_coeff={P.HIGH: fx(pp["coeff"][0]), P.LOW: fx(pp["coeff"][1])})
    return {"profiles": profiles, "gpus": gpus, "queue": q, "cand": cprof, "now": now,
            "predictor": api.InterferencePredictor(params)}
