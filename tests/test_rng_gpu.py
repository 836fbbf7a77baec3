"""GPU: the on-device workload generator (csrc/strait_rng.cuh,
csrc/strait_workload.cu) reproduces numpy 2.3's streams draw for draw, and a
replay batch generated on the device has exactly the inputs (event-ordered
arrivals, per-model index lists, batch noise) of the host path — hence the
same replays as the reference."""
import numpy as np
import pytest

from replay_cases import CASES, case_config

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("ent", ([0, 0], [7, 3], [2 ** 40 + 5, 1], [3, 1, 17], [11, 1_000_003]))
def test_device_rng_equals_numpy(cuda, ent):
    from paper_2604_28175_b200.devgen import rng_draws

    n = 300_000
    raw = rng_draws(ent, 2, 2000).view(np.uint64)
    np.testing.assert_array_equal(raw, np.random.default_rng(np.random.SeedSequence(ent)).bit_generator.random_raw(2000))
    np.testing.assert_array_equal(rng_draws(ent, 0, n, scale=1.7),
                                  np.random.default_rng(np.random.SeedSequence(ent)).exponential(1.7, n))
    np.testing.assert_array_equal(rng_draws(ent, 1, n, loc=0.0, scale=0.05),
                                  np.random.default_rng(np.random.SeedSequence(ent)).normal(0.0, 0.05, n))


def _compare(specs):
    from paper_2604_28175_b200.replay import ReplayBatch

    from oracle import oracle

    h = ReplayBatch(specs).host_inputs()
    h["noise"] = oracle.exp(h.pop("noise_z"))  # the host normals -> glibc exp, as the reference's math.exp
    d = ReplayBatch(specs, generate="device").host_inputs()
    for k in ("req_off", "mr_off", "arr_time", "arr_model", "model_req", "noise"):
        np.testing.assert_array_equal(d[k][:len(h[k])], h[k], err_msg=k)
        assert len(d[k]) == max(1, len(h[k])) or len(d[k]) == len(h[k]), k


@pytest.mark.parametrize("name", CASES)
def test_device_workload_equals_host(cuda, name):
    from paper_2604_28175_b200.replay import ReplaySpec

    _compare([ReplaySpec(case_config(name))])


def test_device_workload_c4_grid_and_replay(cuda):
    """A C4-grid slice (mixed loads / HP fractions / seeds) in one batch, then
    the device-generated batch replays to the host-generated batch's results."""
    from paper_2604_28175_b200.configs import c4_grid
    from paper_2604_28175_b200.replay import ReplayBatch, ReplaySpec

    specs = [ReplaySpec(c, s) for c, s in c4_grid(duration=600.0, seeds=2)[::5]]
    _compare(specs)
    a = ReplayBatch(specs).run(metrics=False)
    b = ReplayBatch(specs, generate="device").run(metrics=False)
    for r in range(len(specs)):
        sa, sb = a.replay_slice(r), b.replay_slice(r)
        for k in ("req_status", "req_violated", "dec_gpu", "dec_est_latency", "counters", "pred_state"):
            np.testing.assert_array_equal(sa[k], sb[k], err_msg=f"replay {r}: {k}")
