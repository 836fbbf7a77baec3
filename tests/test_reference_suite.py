"""CPU: the reference's OWN unit tests for the host-side modules of the path
(pkg/tests/test_pcie.py, test_domain.py, test_workload.py — PCIe FIFO link,
ThroughputTimeline / profiles, arrival generators) run unchanged against this
package through an `infersim` alias (tests/ref_shim).  Runs only where the
reference is mounted (the build container); the GPU-dependent reference
modules are covered by the restated GPU tests (test_scheduler_gpu.py,
test_acceptance_gpu.py, test_replay_gpu.py)."""
import os
import subprocess
import sys

import pytest

from conftest import REPO

REF_TESTS = "/root/reference/pkg/tests"


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference tests not mounted")
@pytest.mark.parametrize("module", ["test_pcie", "test_domain", "test_workload"])
def test_reference_suite_against_mirror(module, tmp_path):
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([os.path.join(REPO, "tests", "ref_shim"), REPO, REF_TESTS]))
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(REF_TESTS, f"{module}.py"), "-q",
                        "-p", "no:cacheprovider", "-x"], cwd=tmp_path, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout


# The rest of the reference's scheduler / baseline suites: every test whose
# functions run on the host mirror (early_drop, TaskQueue, AIMD, the runtime
# state, largest_feasible, the baseline policies, the pass driver).  The tests
# that need the device (check_violate / check_meet / PredictivePolicy.propose)
# are restated in tests/test_scheduler_gpu.py.
DEVICE_ONLY = "not TestCheckViolate and not TestCheckMeet and not TestSchedulePass and " \
              "not test_same_early_drop_sets_across_policies"


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference tests not mounted")
@pytest.mark.parametrize("module,select", [("test_scheduler", DEVICE_ONLY), ("test_baselines", DEVICE_ONLY),
                                           ("test_metrics", "TestNearestRank or TestPerturbProfiles")])
def test_reference_host_suites_against_mirror(module, select, tmp_path):
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([os.path.join(REPO, "tests", "ref_shim"), REPO, REF_TESTS]))
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(REF_TESTS, f"{module}.py"), "-q",
                        "-p", "no:cacheprovider", "-k", select], cwd=tmp_path, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/configs"), reason="reference configs not mounted")
@pytest.mark.parametrize("name,case", [("demo.yaml", "demo"), ("overload.yaml", "overload")])
def test_shipped_yaml_configs_load_to_the_golden_inputs(name, case):
    """config.load_config on the reference's shipped YAML gives exactly the
    replay inputs of the restated config the golden replays were made from."""
    import numpy as np

    from paper_2604_28175_b200.config import load_config
    from paper_2604_28175_b200.replay import ReplayBatch, ReplaySpec
    from replay_cases import case_config

    a = ReplayBatch([ReplaySpec(load_config(os.path.join("/root/reference/pkg/configs", name)))]).host_inputs()
    b = ReplayBatch([ReplaySpec(case_config(case))]).host_inputs()
    for k in b:
        if k == "cfg":
            assert bytes(a[k]) == bytes(b[k])
        else:
            np.testing.assert_array_equal(a[k], b[k], err_msg=k)


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src"), reason="reference not mounted")
def test_perturb_profiles_matches_reference():
    """metrics.perturb_profiles draws and clamps exactly as the reference's
    (metrics.py:161-195), value for value."""
    sys.path.insert(0, "/root/reference/pkg/src")
    try:
        import infersim.metrics as RM
        import infersim.profiles as RP
    finally:
        sys.path.remove("/root/reference/pkg/src")
    from paper_2604_28175_b200.metrics import perturb_profiles
    from paper_2604_28175_b200.profiles import default_profiles

    for mag, seed in ((0.0, 0), (10.0, 3), (35.5, 11), (100.0, 2604)):
        want = RM.perturb_profiles(RP.default_profiles(), mag, seed)
        got = perturb_profiles(default_profiles(), mag, seed)
        assert sorted(want) == sorted(got)
        for mid in want:
            for f in ("throughput", "self_compute", "self_memory", "total_latency", "kernel_latency",
                      "transfer_latency"):
                assert [tuple(r) if isinstance(r, (list, tuple)) else r for r in getattr(got[mid], f)] == \
                       [tuple(r) if isinstance(r, (list, tuple)) else r for r in getattr(want[mid], f)], (mid, f)
    with pytest.raises(ValueError):
        perturb_profiles(default_profiles(), 101.0, 0)
