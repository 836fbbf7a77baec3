"""Shared test setup: marker registration, repo on sys.path, oracle build."""
import os
import subprocess
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built _strait.so")


@pytest.fixture(scope="session")
def oracle():
    subprocess.check_call(["make", "-s", "oracle"], cwd=REPO)  # no-op when up to date
    from oracle import oracle as o

    return o


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
        return cache[name]

    return load


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_28175_b200 import _abi

    _abi.lib()  # missing extension must fail, not skip
    return torch.device("cuda")


def sweep_case(golden, case):
    """Rebuild a SweepSoA from the golden sweep fixture."""
    from paper_2604_28175_b200.sweep import SweepSoA

    g = golden("sweep")
    nm, C, G, conc, S = (int(v) for v in g[f"{case}__geom"])
    arrays = {k.split("__in__")[1]: v for k, v in g.items() if k.startswith(f"{case}__in__")}
    return SweepSoA(nm, C, G, conc, S, 100.0, arrays)
