"""GPU: the replay engine at the edges of its geometry, checked against the C
oracle (itself pinned to the reference by tests/test_replay_oracle.py):
an empty replay, more models than warp lanes (40), more GPUs than lanes (48,
the probe-by-probe propose path) with several concurrency limits and batch
sizes up to 16, every policy in one mixed launch, device-generated inputs, and a
wide node with batch sizes up to 40 and the baseline policies."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _profiles(n, seed=7, max_batch=8):
    from paper_2604_28175_b200.domain import PriorityLevel
    from paper_2604_28175_b200.profiles import random_profile

    rng = np.random.default_rng(seed)
    return {f"e{i:02d}": random_profile(rng, f"e{i:02d}", PriorityLevel.HIGH if i % 3 == 0 else PriorityLevel.LOW,
                                        max_batch_size=max_batch) for i in range(n)}


def _cfg(profiles, rates, duration, n_gpus, conc, policy="predictive", seed=0, sigma=0.05):
    from paper_2604_28175_b200 import config as MC

    doc = {"profiles": profiles, "duration_ms": duration, "seed": seed, "n_gpus": n_gpus,
           "concurrency_limit": conc, "policy": policy, "ground_truth": {"noise_sigma": sigma},
           "workload": {m: {"mode": "poisson", "rate": r} for m, r in rates.items()}}
    return MC.config_from_dict(doc)


def _check(specs, oracle, generate="host"):
    from paper_2604_28175_b200.replay import ReplayBatch

    batch = ReplayBatch(specs, generate=generate)
    res = batch.run()
    res.check()
    ores = oracle.replay(ReplayBatch(specs) if generate == "device" else batch, threads=4)
    for r in range(batch.R):
        d, o = res.replay_slice(r), ores.replay_slice(r)
        assert len(d["dec_time"]) == len(o["dec_time"]), f"replay {r}"
        for k in ("req_status", "req_violated", "req_batch", "dec_pass", "dec_model", "dec_size", "dec_gpu",
                  "dec_est_latency", "dec_intf", "req_completion", "fb_predicted", "cap_gpu", "cap_pct"):
            np.testing.assert_array_equal(d[k], o[k], err_msg=f"replay {r}: {k}")
        np.testing.assert_array_equal(d["counters"][6:13], o["counters"][6:13])
        np.testing.assert_array_equal(d["pred_state"], o["pred_state"])
    return res


def test_empty_and_tiny_replays(cuda, oracle):
    from paper_2604_28175_b200.configs import overload
    from paper_2604_28175_b200.replay import ReplaySpec

    specs = [ReplaySpec(overload(0.001), 0), ReplaySpec(overload(2.0), 1), ReplaySpec(overload(300.0), 2)]
    res = _check(specs, oracle)
    assert res.counters[0][12] == 0  # nothing resolved, nothing to resolve


def test_forty_models_more_than_lanes(cuda, oracle):
    from paper_2604_28175_b200.replay import ReplaySpec

    profs = _profiles(40)
    rates = {m: 120.0 + 15 * i for i, m in enumerate(sorted(profs))}
    specs = [ReplaySpec(_cfg(profs, rates, 400.0, 6, 4, seed=s), s) for s in range(2)]
    _check(specs, oracle)


@pytest.mark.parametrize("conc", [2, 4, 8])
def test_48_gpus_probe_path(cuda, oracle, conc):
    from paper_2604_28175_b200.replay import ReplaySpec

    profs = _profiles(12, seed=11, max_batch=16)
    rates = {m: 900.0 for m in profs}
    _check([ReplaySpec(_cfg(profs, rates, 150.0, 48, conc, seed=3), 3)], oracle)


def test_mixed_policies_and_device_inputs(cuda, oracle):
    from paper_2604_28175_b200.configs import overload
    from paper_2604_28175_b200.replay import ReplaySpec

    specs = []
    for i, p in enumerate(("predictive", "temporal", "static", "reactive")):
        specs.append(ReplaySpec(overload(400.0, policy=p), i))
        specs.append(ReplaySpec(overload(300.0, policy=p, n_gpus=3, concurrency_limit=2), 10 + i))
    _check(specs, oracle, generate="device")


def test_predictive_only_kernel_rejects_a_wrong_policy_mask(cuda):
    """args.policies selects the kernel without the baseline policies; a
    replay whose policy contradicts the mask fails with ValueError instead of
    running the wrong policy."""
    import ctypes as C

    from paper_2604_28175_b200 import _device as D
    from paper_2604_28175_b200.replay import ReplayBatch, ReplayResult, ReplaySpec
    from paper_2604_28175_b200.configs import overload

    batch = ReplayBatch([ReplaySpec(overload(200.0, policy="static"))])
    din, dout = batch.device_inputs(), batch.alloc_outputs(device=True)
    args = batch.args(din, dout, D.ptr)
    assert args.policies == 1 << 2
    args.policies = 1  # claims predictive-only
    D.check(D.lib().strait_replay(C.byref(args), D.stream_handle()))
    res = ReplayResult(batch, {k: D.host(v) for k, v in dout.items()})
    with pytest.raises(ValueError):
        res.check()


def test_fixed_geometry_kernel_rejects_a_wrong_uniform_flag(cuda):
    """args.uniform + the 4x4x6 geometry select the fixed-geometry kernel; a
    replay that does not have that geometry fails with ValueError instead of
    running with the wrong strides."""
    import ctypes as C

    from paper_2604_28175_b200 import _device as D
    from paper_2604_28175_b200.configs import overload
    from paper_2604_28175_b200.replay import ReplayBatch, ReplayResult, ReplaySpec

    batch = ReplayBatch([ReplaySpec(overload(200.0)), ReplaySpec(overload(200.0, n_gpus=2))])
    din, dout = batch.device_inputs(), batch.alloc_outputs(device=True)
    args = batch.args(din, dout, D.ptr)
    assert args.uniform == 0
    args.uniform = 1  # wrongly claims every replay has 4 GPUs
    D.check(D.lib().strait_replay(C.byref(args), D.stream_handle()))
    res = ReplayResult(batch, {k: D.host(v) for k, v in dout.items()})
    assert int(res.counters[0, 0]) == 0 and int(res.counters[1, 0]) != 0
    with pytest.raises(ValueError):
        res.check()


def test_wide_node_large_batches_and_baselines(cuda, oracle):
    """A 16-GPU node (64 slots: the CTA-per-replay layout) with batch sizes up
    to 40 (beyond the 32 sizes the CTA propose job covers, so the master warp's
    probe-by-probe search runs inside the CTA kernel), and every baseline
    policy on the same wide node."""
    from paper_2604_28175_b200.replay import ReplaySpec

    profs = _profiles(8, seed=5, max_batch=40)
    rates = {m: 1500.0 for m in profs}
    specs = [ReplaySpec(_cfg(profs, rates, 120.0, 16, 4, seed=4), 4)]
    specs += [ReplaySpec(_cfg(profs, rates, 120.0, 16, 4, policy=p, seed=5 + i), 5 + i)
              for i, p in enumerate(("temporal", "static", "reactive"))]
    _check(specs, oracle)
