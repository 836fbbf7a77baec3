"""Throughput of large overload sweeps (R replays of 3 s) in one launch."""
import ctypes as C
import os
import sys

import torch

sys.path[:0] = [os.path.join(os.path.dirname(__file__), "..", "tests"), os.path.join(os.path.dirname(__file__), "..")]
from replay_cases import overload_doc  # noqa: E402

from paper_2604_28175_b200 import _device as D  # noqa: E402
from paper_2604_28175_b200 import config as MC  # noqa: E402
from paper_2604_28175_b200.replay import ReplayBatch, ReplaySpec  # noqa: E402

for R in [int(x) for x in (sys.argv[1:] or ["2368", "4736"])]:
    b = ReplayBatch([ReplaySpec(MC.config_from_dict(overload_doc(3000)), s) for s in range(R)], generate="device")
    din, dout = b.device_inputs(), b.alloc_outputs(device=True)
    args = b.args(din, dout, D.ptr)
    best = 1e9
    for _ in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        D.check(D.lib().strait_replay(C.byref(args), D.stream_handle()))
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    print(f"R={R} N={b.N} {best:.3f}s {b.N / best / 1e6:.1f}M req/s", flush=True)
    del din, dout, args, b
    torch.cuda.empty_cache()
