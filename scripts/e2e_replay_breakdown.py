"""Where the C4 replay e2e time goes: host batch build, device stream generation, replay, metrics, D2H."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2604_28175_b200.configs import c4_grid  # noqa: E402
from paper_2604_28175_b200.replay import ReplayBatch, ReplaySpec  # noqa: E402

specs = [ReplaySpec(c, s) for c, s in c4_grid()]
fetch = {"counters", "req_status", "req_violated"}
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    b = ReplayBatch(specs, generate="device")
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    res = b.run(metrics=True, fetch=fetch)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"iter {it}: build+devgen {1e3 * (t1 - t0):.1f} ms, run+metrics+D2H {1e3 * (t2 - t1):.1f} ms, N={b.N}")
