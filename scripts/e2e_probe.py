"""Phase timing of the C4 e2e path: ReplayBatch(generate='device').run()."""
import ctypes as C
import os
import sys
import time

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2604_28175_b200 import _device as D  # noqa: E402
from paper_2604_28175_b200.configs import c4_grid  # noqa: E402
from paper_2604_28175_b200.replay import ReplayBatch, ReplaySpec  # noqa: E402

specs = [ReplaySpec(c, s) for c, s in c4_grid()]


def t():
    torch.cuda.synchronize()
    return time.perf_counter()


for it in range(2):
    t0 = t()
    b = ReplayBatch(specs, generate="device")
    t1 = t()
    din = b.device_inputs()
    t2 = t()
    dout = b.alloc_outputs(device=True)
    args = b.args(din, dout, D.ptr)
    t3 = t()
    D.check(D.lib().strait_replay(C.byref(args), D.stream_handle()))
    t4 = t()
    import numpy as np

    din["window_ms"] = D.dev(np.array([s.config.goodput_window_ms for s in b.specs], dtype=np.float64))
    mout = b.alloc_metrics()
    margs = b.metrics_args(din, dout, mout, D.ptr)
    D.check(D.lib().strait_replay_metrics(C.byref(margs), D.stream_handle()))
    t5 = t()
    x = [D.host(dout[k]) for k in ("counters", "req_status", "req_violated")]
    t6 = t()
    print(f"iter {it}: build+devgen {1e3*(t1-t0):.1f} ms, device_inputs {1e3*(t2-t1):.1f}, alloc {1e3*(t3-t2):.1f}, "
          f"replay {1e3*(t4-t3):.1f}, metrics {1e3*(t5-t4):.1f}, d2h {1e3*(t6-t5):.1f}", flush=True)
