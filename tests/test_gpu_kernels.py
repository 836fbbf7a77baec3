"""GPU parity: the CUDA kernels (through the C-ABI) against the reference's
golden vectors and the C oracle.  Decisions/flags must be identical, and so
must every float: the device exp/log/pow are restatements of the reference
host's glibc routines (csrc/strait_libm.cuh), so the north_star's 1e-5
relative bound is checked but bit-identity is what is required."""
import ctypes as C
import os

import numpy as np
import pytest
import torch

from conftest import sweep_case

pytestmark = pytest.mark.gpu

REL = 1e-5  # north_star tolerance for float latency predictions


def assert_close_bits(got, want, rel=REL, what=""):
    """Within `rel` (north_star) AND bit-identical, NaNs matching."""
    got, want = np.asarray(got), np.asarray(want)
    both_nan = np.isnan(got) & np.isnan(want)
    ok = both_nan | (got == want) | (np.abs(got - want) <= rel * np.maximum(np.abs(want), 1e-300))
    assert ok.all(), f"{what}: {np.count_nonzero(~ok)} values beyond {rel} rel"
    exact = both_nan | (got == want)
    assert exact.all(), f"{what}: {np.count_nonzero(~exact)} of {got.size} values not bit-identical"


def test_predict_vs_golden(cuda, golden):
    from paper_2604_28175_b200.predictor import PredictorParams, predict_parts_batch

    g = golden("predict")
    n = len(g["intf"])
    xs, effs, intfs, sats = [], [], [], []
    for i0 in range(0, n, 100):
        sl = slice(i0, i0 + 100)
        p = PredictorParams(weights=(0.0,) * 5)
        p.apply_vector(list(g["params"][i0]))
        x, eff, intf, sat = predict_parts_batch(p, g["coloc"][sl], g["self_cmp"][sl], g["self_mem"][sl],
                                                g["prio"][sl])
        xs.append(x), effs.append(eff), intfs.append(intf), sats.append(sat)
    np.testing.assert_array_equal(np.concatenate(xs), g["exponent"])  # pure +,* : bit-exact
    np.testing.assert_array_equal(np.concatenate(sats), g["saturated"])
    assert_close_bits(np.concatenate(effs), g["effect"], what="effect")
    assert_close_bits(np.concatenate(intfs), g["intf"], what="intf")


def test_estimate_latency_vs_golden(cuda, golden):
    from paper_2604_28175_b200.predictor import PredictorParams, estimate_latency_batch

    g = golden("latency")
    got = []
    for i in range(len(g["latency"])):
        p = PredictorParams(weights=(0.0,) * 5)
        p.apply_vector(list(g["params"][i]))
        lat, _ = estimate_latency_batch(p, [g["assumed"][i]], g["cmp"][i], g["mem"][i], g["prio"][i], g["total"][i],
                                        g["kernel"][i], g["t_avail"][i], g["front"][i], g["now"][i])
        got.append(lat[0])
    assert_close_bits(got, g["latency"][: len(got)], what="latency")


def test_twa_vs_golden(cuda, golden):
    from paper_2604_28175_b200 import _device as D

    g = golden("twa")
    n = len(g["t0"])
    t0, tl, vl, acc, end = (D.dev(g[k]) for k in ("t0", "t_last", "v_last", "acc", "end"))
    out = D.empty((5, n))
    D.check(D.lib().strait_twa(5, D.ptr(t0), D.ptr(tl), D.ptr(vl), D.ptr(acc), D.ptr(end), n, D.ptr(out),
                               D.stream_handle()))
    np.testing.assert_array_equal(D.host(out), g["twa"])  # +,*,/ only: bit-exact


@pytest.mark.parametrize("stream", ["converge", "adversarial", "edge"])
def test_refit_vs_golden(cuda, golden, stream):
    from paper_2604_28175_b200.predictor import FeedbackSample, InterferencePredictor
    from paper_2604_28175_b200.domain import PriorityLevel

    g = golden("refit")
    tw = g[f"{stream}_twa"]
    samples = [FeedbackSample("b", tuple(tw[:, i]), g[f"{stream}_cmp"][i], g[f"{stream}_mem"][i],
                              PriorityLevel(int(g[f"{stream}_prio"][i])), g[f"{stream}_actual"][i])
               for i in range(tw.shape[1]) if g[f"{stream}_actual"][i] > 0]
    assert len(samples) == tw.shape[1]
    pred = InterferencePredictor()
    res = pred.update_batch(samples)
    traj = g[f"{stream}_traj"]
    got_state = np.array(pred.params.to_vector() + pred.opt.m + pred.opt.v)
    assert pred.opt.step == traj[-1, -1]
    assert_close_bits(got_state, traj[-1, :-1], what="final state")
    np.testing.assert_array_equal([r.skipped for r in res], g[f"{stream}_skipped"])
    np.testing.assert_array_equal([r.saturated for r in res], g[f"{stream}_saturated"])
    assert_close_bits([r.predicted for r in res], g[f"{stream}_predicted"], what="predicted")


def _golden_sweep_check(golden, case, pname, vname, uv, um, path):
    from paper_2604_28175_b200 import sweep as SW

    g = golden("sweep")
    soa = sweep_case(golden, case)
    os.environ["STRAIT_SWEEP_PATH"] = path
    try:
        out = SW.sweep(soa, g[f"{case}__{pname}__params"], use_violate=uv, use_meet=um)
        used = SW.last_sweep_path()
    finally:
        os.environ.pop("STRAIT_SWEEP_PATH", None)
    pre = f"{case}__{pname}__{vname}__"
    np.testing.assert_array_equal(out["pair_flags"], g[pre + "pair_flags"])
    np.testing.assert_array_equal(out["seg_gpu"], g[pre + "seg_gpu"])
    for k in ("pair_latency", "pair_intf", "seg_latency", "seg_intf"):
        assert_close_bits(out[k], g[pre + k], what=k)
    return used


@pytest.mark.parametrize("case", ["c3", "small", "odd"])
@pytest.mark.parametrize("pname", ["default", "strong"])
@pytest.mark.parametrize("path", ["1", "0"])
def test_sweep_vs_golden(cuda, golden, case, pname, path):
    variants = [("full", True, True)]
    if case == "small":
        variants += [("no_meet", True, False), ("no_violate", False, True)]
    for vname, uv, um in variants:
        used = _golden_sweep_check(golden, case, pname, vname, uv, um, path)
        if path == "1":
            assert used == "sync"
        elif case == "c3":
            assert used == "tma-tensor"


@pytest.mark.parametrize("gpus,slots,segs", [(64, 4, 2048), (16, 4, 4096), (8, 8, 1024), (4, 4, 8000),
                                             (32, 2, 777), (1, 1, 5000)])
@pytest.mark.parametrize("path", ["1", "0", "3"])
def test_sweep_vs_oracle_random(cuda, oracle, gpus, slots, segs, path):
    from paper_2604_28175_b200 import sweep as SW
    from paper_2604_28175_b200.microbench import c3_round

    soa = c3_round(11, n_segments=segs, gpus=gpus, slots=slots, concurrency_limit=slots + 1)
    P = np.array([0.3, 2.4, -0.3, 0.3, 0.25, 0.3, 0.2, 0.3, 0.25, 0.2, 0.6, 1.0])
    want = oracle.sweep(soa, P, threads=8)
    os.environ["STRAIT_SWEEP_PATH"] = path
    try:
        got = SW.sweep(soa, P)
    finally:
        os.environ.pop("STRAIT_SWEEP_PATH", None)
    np.testing.assert_array_equal(got["pair_flags"], want["pair_flags"])
    np.testing.assert_array_equal(got["seg_gpu"], want["seg_gpu"])
    for k in ("pair_latency", "pair_intf", "seg_latency", "seg_intf"):
        assert_close_bits(got[k], want[k], what=k)
    assert (want["seg_gpu"] >= 0).any() and (want["seg_gpu"] < 0).any()


def test_round_equals_sweep_plus_refit(cuda, oracle):
    """strait_round (fused launch) == strait_sweep then strait_refit."""
    from paper_2604_28175_b200 import _device as D
    from paper_2604_28175_b200 import sweep as SW
    from paper_2604_28175_b200.microbench import c3_feedback, c3_round
    from paper_2604_28175_b200.predictor import InterferencePredictor

    soa = c3_round(5, n_segments=1024).to_device()
    fb = c3_feedback(5)
    pred = InterferencePredictor()
    P = pred.params.device_vector()
    ref_out = SW.alloc_outputs(soa)
    SW.launch_sweep(soa, P, ref_out)
    state, step = pred.device_state()
    dfb = {k: D.dev(v, torch.int8 if k == "prio" else torch.float64) for k, v in fb.items()}
    args, bc = pred.refit_args(state, step, len(fb["actual"]), dfb["twa"], dfb["self_cmp"], dfb["self_mem"],
                               dfb["prio"], dfb["actual"])
    D.check(D.lib().strait_refit(C.byref(args), D.stream_handle()))
    state2, step2 = pred.device_state()
    args2, _ = pred.refit_args(state2, step2, len(fb["actual"]), dfb["twa"], dfb["self_cmp"], dfb["self_mem"],
                               dfb["prio"], dfb["actual"], bc=bc)
    out = SW.alloc_outputs(soa)
    SW.launch_round(soa, P, out, args2)
    torch.cuda.synchronize()
    for k in out:
        assert torch.equal(out[k].nan_to_num(-7.0), ref_out[k].nan_to_num(-7.0)), k
    assert torch.equal(state, state2) and torch.equal(step, step2)
    # and the refit agrees with the oracle chain
    ostate, ostep, _, _, _ = oracle.refit(pred.params.to_vector() + pred.opt.m + pred.opt.v, 0, fb, nm=5)
    assert_close_bits(D.host(state2), ostate, what="round refit")
    assert int(D.host(step2)[0]) == ostep


def test_errors_map_to_reference_exceptions(cuda):
    from paper_2604_28175_b200.predictor import PredictorParams, predict_interference

    with pytest.raises(ValueError, match="metrics"):
        predict_interference(PredictorParams(), (0.1, 0.2), 0.0, 0.0, 0)


def test_launch_counter_moves(cuda):
    from paper_2604_28175_b200 import _abi
    from paper_2604_28175_b200.predictor import PredictorParams, predict_interference

    before = _abi.lib().strait_kernel_launches()
    predict_interference(PredictorParams(), (0.1,) * 5, 0.2, 0.3, 1)
    assert _abi.lib().strait_kernel_launches() == before + 1


def test_sweep_expand_profile_indexed_snapshot(cuda):
    """A profile-indexed C3 snapshot expanded on the device (strait_sweep_expand)
    is bit-identical to the field-by-field export, and sweeps to the same
    decisions (the e2e path of bench.py)."""
    import torch

    from paper_2604_28175_b200 import _device as D
    from paper_2604_28175_b200 import sweep as SW
    from paper_2604_28175_b200.microbench import c3_compact, c3_round

    soa = c3_round(3, n_segments=512)
    full = soa.to_device()
    comp = c3_compact(soa)
    blank = soa.like({k: (np.zeros_like(v) if v.dtype != np.int8 else np.zeros_like(v)) for k, v in soa.arrays.items()})
    dev = blank.to_device()
    tables = {k: D.dev(v, torch.int8 if v.dtype == np.int8 else torch.float64) for k, v in comp["tables"].items()}
    rows = {k: torch.from_numpy(comp["fields"][k]) for k in ("ent_row", "cand_row")}
    dev_rows = {k: D.empty(len(v), torch.int16) for k, v in rows.items()}
    fields = {k: torch.from_numpy(v) for k, v in comp["fields"].items() if k not in rows}
    SW.load_compact(dev, fields, rows, dev_rows, tables, comp["table_stride"])
    for k in full.arrays:
        np.testing.assert_array_equal(D.host(dev.arrays[k]), D.host(full.arrays[k]), err_msg=k)
    P = D.dev(np.array([0.1, np.e, 0.0] + [0.1] * 5 + [0.1, 0.1, 0.5, 1.0]))
    o1, o2 = SW.alloc_outputs(full), SW.alloc_outputs(dev)
    SW.launch_sweep(full, P, o1)
    SW.launch_sweep(dev, P, o2)
    for k in o1:
        np.testing.assert_array_equal(D.host(o1[k]), D.host(o2[k]), err_msg=k)
