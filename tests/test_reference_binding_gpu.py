"""INTEGRATION.md Level 2 executed on the device: the unmodified reference
simulator (pip-installed into baseline/_ref) with the B200 predictor injected
and with the B200 policy + runtime records behind its registry must
reproduce the stock reference run's trace hash.  Runs in a subprocess (the
CPU suite aliases `infersim` to this package through tests/ref_shim).
Skipped where baseline/_ref was not installed."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not os.path.isdir(os.path.join(REPO, "baseline", "_ref", "infersim")),
                    reason="reference not installed into baseline/_ref")
def test_reference_simulator_with_b200_seams(cuda):
    out = subprocess.run([sys.executable, os.path.join(REPO, "scripts", "reference_binding.py"), "300"],
                         capture_output=True, text=True, timeout=600, cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["estimator_injection"]["match"], res
    assert res["estimator_injection"]["refit_steps"] > 0
    assert res["policy_seam"].get("match"), res
    assert res["policy_seam"]["device_proposes"] > 0
