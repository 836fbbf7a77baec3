"""INTEGRATION.md Level 2, executed: the UNMODIFIED reference simulator
(`infersim`, pip-installed into baseline/_ref, which travels to the GPU box)
with the B200 path bound at its two plugin seams, compared with the stock
reference run of the same config.

  1. estimator injection (simulation.py:123-127,155):
     infersim.simulation.Simulation(cfg, predictor=<B200 InterferencePredictor>)
     -> every completion's refit runs on the device (strait_refit).
  2. policy registry (baselines.py:136-160) + runtime records: make_policy
     routed to "predictive_b200" (one strait_node_propose launch per
     propose) over the B200 GpuRuntimeState / AimdState node records, with the
     pass driver, submit_plan and complete_batch of this package; the event
     loop, queues' arrivals, ground truth, noise and outputs stay the
     reference's own code.

Each run's trace.csv SHA-256 must equal the stock reference run's.

    python scripts/reference_binding.py [duration_ms]   -> one JSON line
"""
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "baseline", "_ref")


def main():
    dur = float(sys.argv[1]) if len(sys.argv) > 1 else 800.0
    if not os.path.isdir(os.path.join(REF, "infersim")):
        print(json.dumps({"unavailable": "baseline/_ref/infersim missing (pip install --target baseline/_ref "
                                         "the reference package first)"}))
        return
    sys.path[:0] = [REF, REPO]
    import infersim
    import infersim.simulation as ref_sim
    from infersim.config import config_from_dict

    import paper_2604_28175_b200 as b200
    from paper_2604_28175_b200 import baselines as b_base
    from paper_2604_28175_b200 import runtime as b_rt
    from paper_2604_28175_b200 import scheduler as b_sch

    sys.path.insert(0, os.path.join(REPO, "tests"))
    from replay_cases import overload_doc

    cfg = config_from_dict(overload_doc(dur))
    out = {"reference": os.path.relpath(infersim.__file__, REPO), "config": f"overload.yaml, {dur:g} ms, seed 0"}

    t0 = time.perf_counter()
    stock = ref_sim.Simulation(cfg).run()
    out["stock"] = {"trace_sha256": stock.trace_hash(), "s": time.perf_counter() - t0,
                    "requests": len(stock.request_rows), "batches": len(stock.batch_rows)}

    # 1. estimator injection: the reference's policy predicts with the injected
    # object's params; its update() is the device refit
    t0 = time.perf_counter()
    pred = b200.InterferencePredictor(b200.PredictorParams(weights=(0.1,) * 5))
    inj = ref_sim.Simulation(cfg, predictor=pred).run()
    out["estimator_injection"] = {"trace_sha256": inj.trace_hash(), "s": time.perf_counter() - t0,
                                  "refit_steps": pred.opt.step, "match": inj.trace_hash() == stock.trace_hash()}

    # 2. the policy seam: what a maintainer adds to infersim's make_policy, plus
    # the runtime records the B200 policy reads in place
    ref_make_policy = ref_sim.make_policy
    calls = {"propose": 0}

    def make_policy(name, predictor, variant="full"):
        if name == "predictive_b200":
            pol = b_base.make_policy("predictive", predictor, variant)
            inner = pol.propose

            def propose(queue, gpus, now):
                calls["propose"] += 1
                return inner(queue, gpus, now)

            pol.propose = propose
            return pol
        return ref_make_policy(name, predictor, variant)

    patched = {"make_policy": make_policy, "GpuRuntimeState": b_rt.GpuRuntimeState, "AimdState": b_rt.AimdState,
               "TaskQueue": b_sch.TaskQueue, "submit_plan": b_sch.submit_plan,
               "complete_batch": b_sch.complete_batch, "run_scheduling_pass": b_sch.run_scheduling_pass}
    saved = {k: getattr(ref_sim, k) for k in patched}
    try:
        for k, v in patched.items():
            setattr(ref_sim, k, v)
        cfg2 = config_from_dict({**overload_doc(dur), "policy": "predictive"})
        cfg2.policy = "predictive_b200"
        t0 = time.perf_counter()
        try:
            pol = ref_sim.Simulation(cfg2, predictor=b200.InterferencePredictor(
                b200.PredictorParams(weights=(0.1,) * 5))).run()
            out["policy_seam"] = {"trace_sha256": pol.trace_hash(), "s": time.perf_counter() - t0,
                                  "device_proposes": calls["propose"], "match": pol.trace_hash() == stock.trace_hash()}
        except Exception as e:  # report, do not hide
            out["policy_seam"] = {"error": f"{type(e).__name__}: {e}"}
    finally:
        for k, v in saved.items():
            setattr(ref_sim, k, v)
    out["ok"] = bool(out["estimator_injection"]["match"] and out["policy_seam"].get("match"))
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
