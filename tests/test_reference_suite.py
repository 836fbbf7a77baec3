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
