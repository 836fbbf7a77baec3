"""Generate the golden fixtures in tests/golden/ by running the REFERENCE
(`infersim`, imported read-only from /root/reference/pkg/src) on seeded
inputs.  The fixtures pin the CPU oracle (oracle/) and the CUDA path.

    python tests/golden/gen_golden.py            # all fixtures
    python tests/golden/gen_golden.py replay     # only the replay fixtures
    python tests/golden/gen_golden.py replay ov_static ...   # selected replay cases

Run in the build container (the reference does not exist on the GPU box;
the committed .npz files travel instead).
"""
from __future__ import annotations

import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, REPO)

from infersim.domain import Batch, PriorityLevel, Request, ThroughputTimeline  # noqa: E402
from infersim.predictor import (FeedbackSample, InterferencePredictor, PredictorParams, kernel_effect,  # noqa: E402
                                predict_interference, pressure_exponent)
from infersim.profiles import random_profile  # noqa: E402
from infersim.runtime import GpuRuntimeState, RunningTaskEntry  # noqa: E402
from infersim.scheduler import check_meet, check_violate  # noqa: E402


def params_vec(p: PredictorParams):
    return np.asarray(p.to_vector(), dtype=np.float64)


def random_params(rng, nm=5):
    return PredictorParams(
        scale=float(rng.uniform(0.01, 2.0)), base=float(rng.uniform(1.1, 4.0)),
        offset=float(rng.uniform(-1.0, 1.0)), weights=tuple(float(w) for w in rng.uniform(-0.5, 0.8, nm)),
        self_compute_weight=float(rng.uniform(-0.5, 0.8)), self_memory_weight=float(rng.uniform(-0.5, 0.8)),
        priority_coeff={PriorityLevel.HIGH: float(rng.uniform(0.1, 1.0)),
                        PriorityLevel.LOW: float(rng.uniform(0.5, 2.0))},
    )


def gen_predict():
    """c01-style draws (test_acceptance.py:96-138): 100 parameter sets x 100
    inputs, plus saturation / clamp edge cases."""
    rng = np.random.default_rng(1)
    P, A, CM, ME, PR, X, EFF, INTF, SAT = [], [], [], [], [], [], [], [], []
    for _ in range(100):
        p = random_params(rng)
        for j in range(100):
            scale_in = 2.5 if j < 90 else 400.0  # a few far-out inputs saturate (z > 500 / inner >= cap)
            a = tuple(float(v) for v in rng.uniform(0.0, scale_in, 5))
            c, m = float(rng.uniform(0, 1)), float(rng.uniform(0, 1))
            pr = PriorityLevel(int(rng.integers(0, 2)))
            x = pressure_exponent(p, a, c, m)
            from infersim.predictor import _raw_effect
            _, sat = _raw_effect(p, x)
            P.append(params_vec(p)); A.append(a); CM.append(c); ME.append(m); PR.append(int(pr))
            X.append(x); EFF.append(kernel_effect(p, x)); INTF.append(predict_interference(p, a, c, m, pr))
            SAT.append(sat)
    np.savez_compressed(os.path.join(HERE, "predict.npz"), params=np.array(P), coloc=np.array(A),
                        self_cmp=np.array(CM), self_mem=np.array(ME), prio=np.array(PR, np.int8),
                        exponent=np.array(X), effect=np.array(EFF), intf=np.array(INTF), saturated=np.array(SAT))


def gen_latency():
    from infersim.pcie import PcieLinkState
    from infersim.predictor import estimate_latency
    from infersim.profiles import default_profiles
    rng = np.random.default_rng(11)
    profiles = list(default_profiles().values())
    rows = {k: [] for k in ("params", "assumed", "cmp", "mem", "prio", "total", "kernel", "t_avail", "front",
                            "now", "latency")}
    for _ in range(2000):
        p = random_params(rng)
        prof = profiles[int(rng.integers(0, len(profiles)))]
        k = int(rng.integers(1, 9))
        now = float(rng.uniform(0, 1000))
        link = PcieLinkState(t_available=now + float(rng.uniform(-5, 5)))
        front = now - float(rng.uniform(0, 10))
        assumed = tuple(float(v) for v in rng.uniform(0, 1.5, 5))
        lat = estimate_latency(p, prof, k, front, link, now, assumed)
        for key, val in (("params", params_vec(p)), ("assumed", assumed), ("cmp", prof.self_compute_at(k)),
                         ("mem", prof.self_memory_at(k)), ("prio", int(prof.priority)),
                         ("total", prof.total_latency_ms(k)), ("kernel", prof.kernel_latency_ms(k)),
                         ("t_avail", link.t_available), ("front", front), ("now", now), ("latency", lat)):
            rows[key].append(val)
    np.savez_compressed(os.path.join(HERE, "latency.npz"), **{k: np.array(v) for k, v in rows.items()})


def gen_refit():
    """Three sequential update streams through InterferencePredictor.update:
    c07-style noisy convergence, adversarial floors (test_predictor.py:392-410)
    and a stream with saturating / non-finite samples."""
    out = {}
    hidden = PredictorParams(scale=0.35, base=2.3, offset=-0.15, weights=(0.22, 0.28, 0.18, 0.25, 0.2),
                             self_compute_weight=0.3, self_memory_weight=0.15,
                             priority_coeff={PriorityLevel.HIGH: 0.6, PriorityLevel.LOW: 1.0})
    for name, seed, n in (("converge", 7, 3000), ("adversarial", 5, 2000), ("edge", 9, 400)):
        rng = np.random.default_rng(seed)
        pred = InterferencePredictor()
        tw, cm, me, pr, ac = [], [], [], [], []
        res_p, res_r, res_s, res_sat, traj = [], [], [], [], []
        for i in range(n):
            if name == "converge":
                agg = tuple(float(a) for a in rng.uniform(0.0, 2.0, 5))
                c, m = float(rng.uniform(0.1, 0.9)), float(rng.uniform(0.1, 0.9))
                p = PriorityLevel.HIGH if rng.uniform() < 0.4 else PriorityLevel.LOW
                truth = predict_interference(hidden, agg, c, m, p)
                actual = 1.0 + (truth - 1.0) * math.exp(float(rng.normal(0.0, 0.05)))
            elif name == "adversarial":
                agg = tuple(float(a) for a in rng.uniform(0, 2, 5))
                c, m = float(rng.uniform(0, 1)), float(rng.uniform(0, 1))
                p = PriorityLevel(int(rng.integers(0, 2)))
                actual = float(rng.uniform(0.2, 6.0))
            else:
                big = i % 7 == 3
                agg = tuple(float(a) for a in rng.uniform(0, 60.0 if big else 2.0, 5))
                c, m = float(rng.uniform(0, 1)), float(rng.uniform(0, 1))
                p = PriorityLevel(int(rng.integers(0, 2)))
                actual = math.inf if i % 11 == 5 else float(rng.uniform(0.5, 8.0))
            r = pred.update(FeedbackSample("b", agg, c, m, p, actual))
            tw.append(agg); cm.append(c); me.append(m); pr.append(int(p)); ac.append(actual)
            res_p.append(r.predicted); res_r.append(r.residual); res_s.append(r.skipped); res_sat.append(r.saturated)
            traj.append(pred.params.to_vector() + pred.opt.m + pred.opt.v + [pred.opt.step])
        out.update({f"{name}_twa": np.array(tw).T.copy(), f"{name}_cmp": np.array(cm), f"{name}_mem": np.array(me),
                    f"{name}_prio": np.array(pr, np.int8), f"{name}_actual": np.array(ac),
                    f"{name}_predicted": np.array(res_p), f"{name}_residual": np.array(res_r),
                    f"{name}_skipped": np.array(res_s), f"{name}_saturated": np.array(res_sat),
                    f"{name}_traj": np.array(traj)})
    init = InterferencePredictor()
    out["init_state"] = np.array(init.params.to_vector() + init.opt.m + init.opt.v)
    np.savez_compressed(os.path.join(HERE, "refit.npz"), **out)


def rebuild_pair(soa, p, profiles_by_idx):
    """Reference GpuRuntimeState for pair p of the SoA (object-level rebuild)."""
    nm, Cs = soa.n_metrics, soa.n_slots
    g = p % soa.gpus_per_segment
    gpu = GpuRuntimeState(g, nm, soa.concurrency_limit)
    nrun = int(soa.arrays["gpu_n_running"][p])
    Tn = soa.n_triples
    for c in range(nrun):
        t = p * Cs + c
        prio = PriorityLevel(int(soa.arrays["ent_prio"][t]))
        req = Request(f"r{t}", "m", soa.now - 50.0, soa.now + 1000.0)
        batch = Batch(f"b{t}", "m", 1, prio, req.arrival_time, [req])
        twa = tuple(float(soa.arrays["ent_twa"][m, t]) for m in range(nm))
        e = RunningTaskEntry(
            batch=batch,
            contribution=tuple(float(soa.arrays["ent_contrib"][m, t]) for m in range(nm)),
            self_compute=float(soa.arrays["ent_self_cmp"][t]), self_memory=float(soa.arrays["ent_self_mem"][t]),
            kernel_latency_ms=float(soa.arrays["ent_t_kernel"][t]),
            deadline_abs=float(soa.arrays["ent_deadline_abs"][t]), intf_predicted=1.0,
            kernel_start_estimate=float(soa.arrays["ent_kstart"][t]),
            timeline=ThroughputTimeline([(soa.now, twa)]),  # TWA(now) == twa exactly (total <= 0 branch)
        )
        gpu.running.append(e)
    gpu._recompute_aggregate()
    agg = np.array(gpu.aggregate_throughput)
    assert np.array_equal(agg, soa.arrays["gpu_agg"][:, p]), "generator aggregate != reference list-order sum"
    assert np.array_equal(np.array(gpu.low_priority_aggregate()), soa.arrays["gpu_lp_agg"][:, p])
    gpu.aimd.cap_pct = float(soa.arrays["gpu_cap_pct"][p])
    gpu.pcie.t_available = float(soa.arrays["gpu_t_avail"][p])
    del Tn
    return gpu


def reference_sweep(soa, pred, ref_profiles, use_violate=True, use_meet=True):
    """best_for (scheduler.py:263-280) on rebuilt objects for every segment."""
    S, G = soa.n_segments, soa.gpus_per_segment
    flags = np.zeros(S * G, np.uint8)
    plat = np.full(S * G, np.nan)
    pintf = np.full(S * G, np.nan)
    sg = np.full(S, -1, np.int32)
    sl = np.full(S, np.nan)
    si = np.full(S, np.nan)
    for s in range(S):
        prof = ref_profiles[int(soa.meta["cand_model"][s])]
        k = int(soa.meta["cand_size"][s])
        front = float(soa.arrays["cand_front"][s])
        best = None
        for g in range(G):
            p = s * G + g
            gpu = rebuild_pair(soa, p, ref_profiles)
            if not gpu.has_slot():
                continue
            f = 1
            v = check_violate(gpu, prof, k, soa.now, pred)
            ok, lat, intf, _ = check_meet(gpu, prof, k, front, soa.now, pred)
            f |= (2 if v else 0) | (4 if ok else 0)
            admitted = not (use_violate and v) and not (use_meet and not ok)
            if admitted:
                f |= 8
                if best is None or (lat, g) < (best[0], best[1]):
                    best = (lat, g, intf)
            flags[p], plat[p], pintf[p] = f, lat, intf
        if best is not None:
            sl[s], sg[s], si[s] = best
    return dict(pair_flags=flags, pair_latency=plat, pair_intf=pintf, seg_gpu=sg, seg_latency=sl, seg_intf=si)


def gen_sweep():
    from paper_2604_28175_b200.microbench import c3_round
    rng = np.random.default_rng(2604)
    ref_profiles = [random_profile(rng, f"m{i:02d}", PriorityLevel.HIGH if i < 8 else PriorityLevel.LOW)
                    for i in range(32)]
    from paper_2604_28175_b200.profiles import profile_to_dict
    from infersim.profiles import profile_to_dict as ref_to_dict
    from paper_2604_28175_b200.microbench import c3_profiles
    assert [profile_to_dict(p) for p in c3_profiles()] == [ref_to_dict(p) for p in ref_profiles]
    cases = {
        "c3": dict(round_idx=0, n_segments=48, gpus=64, slots=4),
        "small": dict(round_idx=1, n_segments=300, gpus=4, slots=4),
        "odd": dict(round_idx=2, n_segments=111, gpus=3, slots=4),
    }
    preds = {
        "default": InterferencePredictor(),
        "strong": InterferencePredictor(PredictorParams(scale=0.5, base=2.6, offset=-0.4,
                                                        weights=(0.3, 0.25, 0.35, 0.2, 0.3),
                                                        self_compute_weight=0.25, self_memory_weight=0.2)),
    }
    out = {}
    for cname, kw in cases.items():
        soa = c3_round(profiles=None, **kw)
        for k, v in soa.arrays.items():
            out[f"{cname}__in__{k}"] = v
        for k, v in soa.meta.items():
            out[f"{cname}__meta__{k}"] = v
        out[f"{cname}__geom"] = np.array([soa.n_metrics, soa.n_slots, soa.gpus_per_segment, soa.concurrency_limit,
                                          soa.n_segments])
        for pname, pred in preds.items():
            out[f"{cname}__{pname}__params"] = params_vec(pred.params)
            variants = [("full", True, True)] + ([("no_meet", True, False), ("no_violate", False, True)]
                                                 if cname == "small" else [])
            for vname, uv, um in variants:
                res = reference_sweep(soa, pred, ref_profiles, uv, um)
                for k, v in res.items():
                    out[f"{cname}__{pname}__{vname}__{k}"] = v
    np.savez_compressed(os.path.join(HERE, "sweep.npz"), **out)


def gen_twa():
    """Random step-hold timelines -> reference time_weighted_average."""
    rng = np.random.default_rng(21)
    rows = {k: [] for k in ("t0", "t_last", "v_last", "acc", "end", "twa", "ns")}
    from paper_2604_28175_b200.domain import ThroughputTimeline as MyTL
    for i in range(3000):
        n = int(rng.integers(1, 9))
        t = 100.0 * rng.uniform()
        ref, mine = ThroughputTimeline(), MyTL()
        for j in range(n):
            if j and rng.uniform() < 0.2:
                pass  # same timestamp -> replace
            else:
                t += float(rng.exponential(1.0))
            v = tuple(float(x) for x in rng.uniform(0, 2, 5))
            ref.record(t, v)
            mine.record(t, v)
        end = t + (0.0 if i % 5 == 0 else float(rng.exponential(2.0)))
        twa = ref.time_weighted_average(end)
        rows["t0"].append(mine.times[0]); rows["t_last"].append(mine.times[-1])
        rows["v_last"].append(mine.values[-1]); rows["acc"].append(mine.acc); rows["end"].append(end)
        rows["twa"].append(twa); rows["ns"].append(len(ref))
    np.savez_compressed(os.path.join(HERE, "twa.npz"),
                        **{k: (np.array(v).T.copy() if k in ("v_last", "acc", "twa") else np.array(v))
                           for k, v in rows.items()})


def gen_lossgrad():
    """Reference loss_gradient on random (params, sample) pairs, including
    clamped and saturated ones, plus a 300-step adam_step trajectory with an
    inactive entry (predictor.py:124-145,271-309)."""
    from infersim.predictor import FeedbackSample, OptimizerState, PredictorParams, adam_step, loss_gradient
    rng = np.random.default_rng(303)
    rows = {k: [] for k in ("P", "twa", "cmp", "mem", "prio", "actual", "pred", "res", "sat", "grad")}
    for i in range(3000):
        p = PredictorParams(scale=float(rng.uniform(0.01, 2.0)), base=float(rng.uniform(1.01, 6.0)),
                            offset=float(rng.uniform(-3.0, 1.0)), weights=tuple(rng.uniform(-0.5, 1.5, 5).tolist()),
                            self_compute_weight=float(rng.uniform(-0.5, 1.0)),
                            self_memory_weight=float(rng.uniform(-0.5, 1.0)),
                            priority_coeff={PriorityLevel.HIGH: float(rng.uniform(0.1, 2.0)),
                                            PriorityLevel.LOW: float(rng.uniform(0.1, 2.0))})
        tw = tuple(rng.uniform(0, 3 if i % 5 else 40, 5).tolist())
        s = FeedbackSample("b", tw, float(rng.uniform()), float(rng.uniform()),
                           PriorityLevel(int(rng.integers(0, 2))), float(rng.uniform(0.5, 8.0)))
        pred, res, sat, grad = loss_gradient(p, s, 0.5)
        rows["P"].append(p.to_vector()); rows["twa"].append(tw); rows["cmp"].append(s.self_compute)
        rows["mem"].append(s.self_memory); rows["prio"].append(int(s.priority)); rows["actual"].append(s.actual)
        rows["pred"].append(pred); rows["res"].append(res); rows["sat"].append(sat); rows["grad"].append(grad)
    out = {k: np.array(v) for k, v in rows.items()}
    n = 12
    opt = OptimizerState(m=[0.0] * n, v=[0.0] * n)
    values = rng.normal(0, 1, n).tolist()
    out["adam_init"] = np.array(values)
    grads = rng.normal(0, 2, (300, n))
    active = [i != 7 for i in range(n)]
    traj = []
    for g in grads:
        adam_step(opt, values, g.tolist(), active=active)
        traj.append(list(values) + list(opt.m) + list(opt.v))
    out["adam_grads"], out["adam_traj"], out["adam_active"] = grads, np.array(traj), np.array(active)
    np.savez_compressed(os.path.join(HERE, "lossgrad.npz"), **out)


def gen_gt():
    """Random (params, co-located aggregate, self terms, priority, noise) ->
    reference ground_truth_slowdown (oracle.py:55-77), both families,
    including clamped (effect <= 0) and large-exponent inputs."""
    from infersim.oracle import GroundTruthParams, ground_truth_slowdown
    rng = np.random.default_rng(77)
    rows = {k: [] for k in ("family", "scale", "base", "offset", "w", "w_cmp", "w_mem", "pf", "co", "cmp", "mem",
                            "prio", "noise", "out")}
    for i in range(4000):
        fam = "exponential" if i % 3 else "quadratic"
        p = GroundTruthParams(family=fam, scale=float(rng.uniform(0.05, 2.0)), base=float(rng.uniform(1.01, 6.0)),
                              offset=float(rng.uniform(-2.0, 0.5)), weights=tuple(rng.uniform(0, 1, 5).tolist()),
                              self_compute_weight=float(rng.uniform(0, 1)), self_memory_weight=float(rng.uniform(0, 1)),
                              priority_factor={PriorityLevel.HIGH: float(rng.uniform(0.2, 1)),
                                               PriorityLevel.LOW: float(rng.uniform(0.5, 1.5))})
        co = rng.uniform(0, 3 if i % 7 else 30, 5).tolist()
        cmp_, mem = float(rng.uniform()), float(rng.uniform())
        pr = PriorityLevel.HIGH if rng.uniform() < 0.5 else PriorityLevel.LOW
        noise = float(np.exp(rng.normal(0, 0.05))) if i % 4 else 1.0
        rows["family"].append(fam == "quadratic"); rows["scale"].append(p.scale); rows["base"].append(p.base)
        rows["offset"].append(p.offset); rows["w"].append(p.weights); rows["w_cmp"].append(p.self_compute_weight)
        rows["w_mem"].append(p.self_memory_weight)
        rows["pf"].append((p.priority_factor[PriorityLevel.HIGH], p.priority_factor[PriorityLevel.LOW]))
        rows["co"].append(co); rows["cmp"].append(cmp_); rows["mem"].append(mem); rows["prio"].append(int(pr))
        rows["noise"].append(noise)
        rows["out"].append(ground_truth_slowdown(p, co, cmp_, mem, pr, noise))
    np.savez_compressed(os.path.join(HERE, "gt.npz"), **{k: np.array(v) for k, v in rows.items()})


# ----------------------------------------------------------------------------- replays
C1_DOC = {"profiles": "default6", "duration_ms": 26316, "seed": 1, "n_gpus": 1, "policy": "predictive",
          "ground_truth": {"noise_sigma": 0.05},
          "workload": {"resnet50": {"mode": "poisson", "rate": 300}, "roberta_b": {"mode": "poisson", "rate": 80}}}
OVERLOAD_GT = {"family": "exponential", "scale": 0.5, "base": 2.718281828459045, "offset": -0.7686,
               "weights": [0.3] * 5, "self_compute_weight": 0.25, "self_memory_weight": 0.2,
               "priority_factor": {"high": 0.6, "low": 1.0}, "noise_sigma": 0.05}
OVERLOAD_WL = {"resnet50": {"mode": "poisson", "rate": 2200}, "vit_b16": {"mode": "poisson", "rate": 800},
               "yolo_v8n": {"mode": "poisson", "rate": 1300}, "convnext_b": {"mode": "poisson", "rate": 650},
               "vgg19": {"mode": "poisson", "rate": 650}, "roberta_b": {"mode": "poisson", "rate": 400}}


def overload_doc(duration, **kw):
    d = {"profiles": "default6", "duration_ms": duration, "seed": 0, "n_gpus": 4, "concurrency_limit": 4,
         "policy": "predictive", "goodput_window_ms": 1000, "ground_truth": dict(OVERLOAD_GT),
         "workload": dict(OVERLOAD_WL)}
    d.update(kw)
    return d


def c5_slice_doc(tmpdir, duration=150):
    """C5 shape: 64 GPUs, 20 random profiles, bursty HP trace + LP Poisson."""
    import infersim.profiles as RP
    rng = np.random.default_rng(2604)
    profs = {f"m{i:02d}": RP.random_profile(rng, f"m{i:02d}", PriorityLevel.HIGH if i < 6 else PriorityLevel.LOW)
             for i in range(20)}
    pdir = os.path.join(tmpdir, "c5_profiles")
    RP.save_profiles_dir(profs, pdir)
    trace = os.path.join(tmpdir, "c5_trace.csv")
    with open(trace, "w") as f:
        f.write("function_id,minute_index,count\n")
        for i in range(6):
            for m in range(2):
                f.write(f"hp{i},{m},{int(rng.lognormal(math.log(150000), 0.6))}\n")
    wl = {f"m{i:02d}": ({"mode": "trace", "trace_file": trace, "function_id": f"hp{i}", "scale": 1.0} if i < 6
                        else {"mode": "poisson", "rate": 2600}) for i in range(20)}
    return {"profiles": pdir, "duration_ms": duration, "seed": 0, "n_gpus": 64, "concurrency_limit": 4,
            "policy": "predictive", "ground_truth": {"noise_sigma": 0.05}, "workload": wl}


REPLAY_CASES = {
    "demo": ("yaml", "/root/reference/pkg/configs/demo.yaml", None),
    "c1": ("doc", C1_DOC, None),
    "overload": ("yaml", "/root/reference/pkg/configs/overload.yaml", None),
    "trace": ("doc", None, "trace"),
    "ov_no_meet": ("doc", overload_doc(500, policy_variant="no_meet"), None),
    "ov_no_violate": ("doc", overload_doc(500, policy_variant="no_violate_aimd"), None),
    "ov_no_prio": ("doc", overload_doc(500, policy_variant="no_priority_scan"), None),
    "ov_no_gamma": ("doc", overload_doc(500, policy_variant="no_gamma_advantage"), None),
    "ov_quadratic": ("doc", overload_doc(500, ground_truth=dict(OVERLOAD_GT, family="quadratic", scale=0.3,
                                                                 offset=-0.4)), None),
    "ov_nonoise_2gpu": ("doc", overload_doc(400, n_gpus=2, ground_truth=dict(OVERLOAD_GT, noise_sigma=0.0)), None),
    "c5_slice": ("doc", None, "c5"),
    # baseline policies behind the same pass seam (baselines.py:40-133)
    "ov_temporal": ("doc", overload_doc(500, policy="temporal"), None),
    "ov_static": ("doc", overload_doc(500, policy="static"), None),
    "ov_reactive": ("doc", overload_doc(1500, policy="reactive"), None),
    "c1_reactive": ("doc", dict(C1_DOC, duration_ms=5000, policy="reactive"), None),
}


def replay_case_docs(name, tmpdir):
    kind, src, special = REPLAY_CASES[name]
    if special == "trace":
        import yaml
        doc = yaml.safe_load(open("/root/reference/pkg/configs/trace_replay.yaml"))
        doc["duration_ms"] = 30000
        return doc, "/root/reference/pkg/configs"
    if special == "c5":
        return c5_slice_doc(tmpdir), tmpdir
    if kind == "yaml":
        import yaml
        return yaml.safe_load(open(src)), os.path.dirname(src)
    return src, "."


def reference_replay_arrays(name, tmpdir):
    import infersim.config as RC
    from infersim.simulation import Simulation, parse_segments
    from paper_2604_28175_b200 import config as MC
    from paper_2604_28175_b200.replay import ReplayBatch, ReplaySpec

    doc, base = replay_case_docs(name, tmpdir)
    rcfg = RC.config_from_dict(doc, base_dir=base)
    mcfg = MC.config_from_dict(doc, base_dir=base)
    sim = Simulation(rcfg)
    res = sim.run()
    batch = ReplayBatch([ReplaySpec(mcfg)])
    ids = batch.tab["ids"]
    mr = batch.inputs["model_req"]
    mr_off = batch.inputs["mr_off"]
    out = {}
    # pin the workload generator: the reference's streams, model-major
    streams = rcfg.workload.generate(rcfg.seed)
    ref_times = np.concatenate([np.asarray(streams.get(m, []), dtype=np.float64) for m in ids])
    my_times = batch.inputs["arr_time"][np.argsort(mr, kind="stable")] if len(mr) else np.empty(0)
    my_model_major = batch.inputs["arr_time"][mr]
    assert np.array_equal(ref_times, my_model_major), f"{name}: workload streams differ"
    del my_times
    N = batch.N
    st = np.zeros(N, np.int8); vi = np.zeros(N, np.uint8); comp = np.full(N, np.nan); rb = np.full(N, -1, np.int32)
    for row in res.request_rows:
        mid, k = row["request"].rsplit("-", 1)
        g = mr[mr_off[ids.index(mid)] + int(k)]
        st[g] = 2 if row["dropped"] else 1
        vi[g] = row["violated"]
        if not row["dropped"]:
            comp[g] = row["completion"]
            rb[g] = int(row["batch"][1:])
    out.update(req_status=st, req_violated=vi, req_completion=comp, req_batch=rb)
    D = res.decision_rows
    out.update(dec_time=np.array([d["time"] for d in D]), dec_pass=np.array([d["pass_id"] for d in D], np.int32),
               dec_model=np.array([ids.index(d["model"]) for d in D], np.int16),
               dec_size=np.array([d["size"] for d in D], np.int8), dec_gpu=np.array([d["gpu"] for d in D], np.int16),
               dec_est_latency=np.array([d["est_latency"] for d in D]),
               dec_intf=np.array([d["intf_pred"] for d in D]))
    nb = len(D)
    cols = {k: np.full(nb, np.nan) for k in ("b_front", "b_transfer_start", "b_kernel_start", "b_kernel_end",
                                              "b_completion", "b_work", "fb_predicted", "fb_actual",
                                              "fb_residual")}
    done = np.full(nb, -1, np.int32)
    flags = np.zeros(nb, np.uint8)
    for j, row in enumerate(res.batch_rows):
        b = int(row["batch"][1:])
        cols["b_front"][b] = row["front_enqueue"]
        cols["b_transfer_start"][b] = row["transfer_start"]
        cols["b_kernel_start"][b] = row["kernel_start"]
        cols["b_kernel_end"][b] = row["kernel_end"]
        cols["b_completion"][b] = row["completion"]
        cols["b_work"][b] = sum(d / s for d, s in parse_segments(row["segments"]))
        done[b] = j
    for row in res.feedback_rows:
        b = int(row["batch"][1:])
        cols["fb_predicted"][b] = row["predicted"]
        cols["fb_actual"][b] = row["actual"]
        cols["fb_residual"][b] = row["residual"]
        flags[b] = (1 if row["skipped"] else 0) | (2 if row["saturated"] else 0)
    out.update(cols)
    out.update(b_done_order=done, fb_flags=flags)
    out.update(cap_time=np.array([c["time"] for c in res.cap_rows]),
               cap_gpu=np.array([c["gpu"] for c in res.cap_rows], np.int16),
               cap_pct=np.array([c["cap_pct"] for c in res.cap_rows]))
    p = sim.predictor
    out["pred_state"] = np.array(p.params.to_vector() + p.opt.m + p.opt.v)
    out["pred_step"] = np.array(p.opt.step)
    m = res.metrics.per_class
    out["class_counts"] = np.array([[m[c].arrivals, m[c].dropped, m[c].violations] for c in PriorityLevel])
    out["trace_hash"] = np.array(res.trace_hash())
    # the reference's own metrics (metrics.py:88-158), window = config.goodput_window_ms
    import json
    out["metrics_json"] = np.array(json.dumps(res.metrics.to_dict()))
    out["goodput_window_ms"] = np.array(rcfg.goodput_window_ms)
    return out


def gen_replay(names=None):
    import tempfile
    import yaml
    os.makedirs(os.path.join(HERE, "replay"), exist_ok=True)
    with tempfile.TemporaryDirectory() as tmp:
        for name in names or REPLAY_CASES:
            arrays = reference_replay_arrays(name, tmp)
            doc, _ = replay_case_docs(name, tmp)
            np.savez_compressed(os.path.join(HERE, "replay", f"{name}.npz"), **arrays)
            print(f"  {name}: {len(arrays['req_status'])} requests, {len(arrays['dec_time'])} batches, "
                  f"classes {arrays['class_counts'].tolist()}", flush=True)


CSV_FILES = ("trace", "requests", "decisions", "feedback", "caps", "batches")


def reference_csv_sha(res):
    """sha256 of each run-directory CSV text the reference writes
    (report.py:92-106, rows_to_csv_text; trace = SimResult.trace_hash)."""
    import hashlib
    from infersim.report import RUN_FILES, rows_to_csv_text
    payload = {"trace": res.trace_rows, "requests": res.request_rows, "decisions": res.decision_rows,
               "feedback": res.feedback_rows, "caps": res.cap_rows, "batches": res.batch_rows}
    out = {k: hashlib.sha256(rows_to_csv_text(payload[k], RUN_FILES[k][1]).encode()).hexdigest() for k in CSV_FILES}
    assert out["trace"] == res.trace_hash()
    return out


def gen_csvsha(seeds=16):
    """tests/golden/replay_csv_sha.json: the reference's CSV fingerprints for
    every golden replay case and for overload.yaml seeds 0..15."""
    import json
    import tempfile
    import yaml
    import infersim.config as RC
    from infersim.simulation import Simulation
    out = {"cases": {}, "overload_seeds": {}}
    with tempfile.TemporaryDirectory() as tmp:
        for name in REPLAY_CASES:
            doc, base = replay_case_docs(name, tmp)
            out["cases"][name] = reference_csv_sha(Simulation(RC.config_from_dict(doc, base_dir=base)).run())
            print(" ", name, out["cases"][name]["trace"][:16], flush=True)
    doc = yaml.safe_load(open("/root/reference/pkg/configs/overload.yaml"))
    for seed in range(seeds):
        cfg = RC.config_from_dict(doc, base_dir="/root/reference/pkg/configs")
        out["overload_seeds"][str(seed)] = reference_csv_sha(Simulation(cfg, seed=seed).run())
        print("  overload seed", seed, out["overload_seeds"][str(seed)]["trace"][:16], flush=True)
    with open(os.path.join(HERE, "replay_csv_sha.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    what = sys.argv[1:] or ["predict", "latency", "refit", "sweep", "twa", "replay"]
    if what[0] == "replay" and len(what) > 1:  # gen_golden.py replay <case> ...
        gen_replay(what[1:])
        sys.exit(0)
    for w in what:
        print("generating", w, flush=True)
        globals()[f"gen_{w}"]()
