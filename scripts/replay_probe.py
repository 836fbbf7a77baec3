"""Replay-engine timing probe (device time of strait_replay vs the C oracle)."""
import os
import sys
import time

import numpy as np
import torch

sys.path[:0] = [os.path.join(os.path.dirname(__file__), "..", "tests"), os.path.join(os.path.dirname(__file__), "..")]
from replay_cases import overload_doc  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_2604_28175_b200 import _device as D  # noqa: E402
from paper_2604_28175_b200 import config as MC  # noqa: E402
from paper_2604_28175_b200.replay import ReplayBatch, ReplaySpec  # noqa: E402
import ctypes as C  # noqa: E402


def timed(batch, reps=2):
    din = batch.device_inputs()
    state0 = din["pred_state"].clone()
    step0 = din["pred_step"].clone()
    dout = batch.alloc_outputs(device=True)
    args = batch.args(din, dout, D.ptr)
    best = 1e9
    for _ in range(reps):
        din["pred_state"].copy_(state0)
        din["pred_step"].copy_(step0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        D.check(D.lib().strait_replay(C.byref(args), D.stream_handle()))
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    cnt = D.host(dout["counters"]).reshape(batch.R, -1)
    assert (cnt[:, 0] == 0).all(), cnt[:, 0]
    return best


def main():
    cases = [("overload 3s x1", [overload_doc(3000)], 1),
             ("overload 30s x1", [overload_doc(30000)], 1),
             ("C2 1M x1", [overload_doc(166667)], 1)]
    for name, docs, _ in cases:
        b = ReplayBatch([ReplaySpec(MC.config_from_dict(d)) for d in docs])
        t = timed(b)
        t0 = time.perf_counter()
        oracle.replay(b)
        tc = time.perf_counter() - t0
        print(f"{name}: N={b.N} device {t:.3f}s ({b.N / t:.0f} req/s)  oracle 1 core {tc:.3f}s ({b.N / tc:.0f} req/s)",
              flush=True)
    for R in (148, 592, 1184, 2368):
        specs = [ReplaySpec(MC.config_from_dict(overload_doc(3000)), s) for s in range(R)]
        b = ReplayBatch(specs)
        t = timed(b)
        print(f"overload 3s x{R}: N={b.N} device {t:.3f}s ({b.N / t:.0f} req/s)", flush=True)


if __name__ == "__main__":
    main()
