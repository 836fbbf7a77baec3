"""Launch ONE strait_replay batch of R overload replays (for ncu captures)."""
import ctypes as C
import os
import sys

import torch

sys.path[:0] = [os.path.join(os.path.dirname(__file__), "..", "tests"), os.path.join(os.path.dirname(__file__), "..")]
from replay_cases import overload_doc  # noqa: E402

from paper_2604_28175_b200 import _device as D  # noqa: E402
from paper_2604_28175_b200 import config as MC  # noqa: E402
from paper_2604_28175_b200.replay import ReplayBatch, ReplaySpec  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 1
DUR = float(sys.argv[2]) if len(sys.argv) > 2 else 3000.0
b = ReplayBatch([ReplaySpec(MC.config_from_dict(overload_doc(DUR)), s) for s in range(R)])
din, dout = b.device_inputs(), b.alloc_outputs(device=True)
args = b.args(din, dout, D.ptr)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
D.check(D.lib().strait_replay(C.byref(args), D.stream_handle()))
e1.record()
torch.cuda.synchronize()
print(f"R={R} N={b.N} {e0.elapsed_time(e1):.1f} ms")
