"""C5-shape single replay (64 GPUs, 20 models): device vs C oracle time."""
import ctypes as C
import os
import sys
import time

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from oracle import oracle  # noqa: E402
from paper_2604_28175_b200 import _device as D  # noqa: E402
from paper_2604_28175_b200.configs import c5  # noqa: E402
from paper_2604_28175_b200.replay import ReplayBatch, ReplaySpec  # noqa: E402

for dur in (150.0, 1000.0):
    b = ReplayBatch([ReplaySpec(c5(duration=dur))], generate="device")
    din, dout = b.device_inputs(), b.alloc_outputs(device=True)
    args = b.args(din, dout, D.ptr)
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        D.check(D.lib().strait_replay(C.byref(args), D.stream_handle()))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    hb = ReplayBatch([ReplaySpec(c5(duration=dur))])
    t0 = time.perf_counter()
    oracle.replay(hb)
    to = time.perf_counter() - t0
    print(f"C5 {dur} ms: N={b.N} device {dt:.3f}s ({b.N / dt:.0f} req/s) oracle {to:.3f}s ({b.N / to:.0f} req/s)",
          flush=True)
