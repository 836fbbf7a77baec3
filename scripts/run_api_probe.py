"""Drop-in API speed: run(config) (traced, rows + CSV-ready) on overload.yaml 3 s."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2604_28175_b200 import run  # noqa: E402
from paper_2604_28175_b200.configs import overload  # noqa: E402

cfg = overload(3000.0)
for i in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = run(cfg)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    h = res.trace_hash()
    t2 = time.perf_counter()
    print(f"run(): {t1 - t0:.3f}s ({17927 / (t1 - t0):.0f} req/s), trace rows + hash {t2 - t1:.3f}s, hash {h[:12]}")
