"""Per-phase cycle accounting of the replay engine (diagnostic build `make prof`):
STRAIT_LIB=build/prof/_strait.so python scripts/replay_profile.py [duration_ms] [load]"""
import ctypes as C
import os
import sys

import numpy as np

sys.path[:0] = [os.path.join(os.path.dirname(__file__), "..", "tests"), os.path.join(os.path.dirname(__file__), "..")]
from replay_cases import overload_doc  # noqa: E402

from paper_2604_28175_b200 import _device as D  # noqa: E402
from paper_2604_28175_b200 import config as MC  # noqa: E402
from paper_2604_28175_b200.configs import c4_point  # noqa: E402
from paper_2604_28175_b200.replay import ReplayBatch, ReplaySpec  # noqa: E402
from paper_2604_28175_b200._replay_abi import RC  # noqa: E402

NAMES = ["select", "arrival", "pass:rank", "pass:early_drop", "pass:eligible+icur_all", "pass:propose",
         "pass:submit", "pass:icur_gpu", "pass:timeouts", "transfer_complete", "kernel_complete(all)",
         "  kc:update", "-", "tick", "post", "TOTAL"]


def main():
    dur = float(sys.argv[1]) if len(sys.argv) > 1 else 3000.0
    cases = [("overload", MC.config_from_dict(overload_doc(dur)))]
    if len(sys.argv) > 2:
        cases.append((f"c4 lambda={sys.argv[2]} f=0.5", c4_point(float(sys.argv[2]), 0.5, dur)))
    if len(sys.argv) > 3:
        from paper_2604_28175_b200.configs import c5
        cases.append((f"c5 {sys.argv[3]} ms (64 GPUs, 20 models)", c5(float(sys.argv[3]))))
    lib = D.lib()
    lib.strait_replay_profile.restype = C.c_int
    cw = np.zeros(48, np.uint64)
    for name, cfg in cases:
        b = ReplayBatch([ReplaySpec(cfg)])
        out = np.zeros(31, np.uint64)
        lib.strait_replay_profile(out.ctypes.data)  # reset
        lib.strait_replay_cta_profile(cw.ctypes.data)
        res = b.run(metrics=False)
        lib.strait_replay_profile(out.ctypes.data)
        c = res.counters[0]
        n = b.N
        tot = float(out[15])
        print(f"== {name}: N={n} events={c[RC['EVENTS']]} passes={c[RC['PASSES']]} batches={c[RC['BATCHES']]}"
              f"  total {tot / 1.965e9 * 1e3:.1f} ms at 1.965 GHz, {tot / n:.0f} cycles/request")
        for i, nm in enumerate(NAMES):
            if nm == "-":
                continue
            print(f"  {nm:26s} {100 * out[i] / tot:5.1f}%  {out[i] / n:8.0f} cyc/req")
        p = c[RC['PASSES']]
        print(f"  per pass: queues visited {out[16] / p:.2f}, eligible {out[17] / p:.2f}, wide proposes "
              f"{out[18] / p:.2f}, submits {out[19] / p:.2f}, icur_all {out[20] / p:.2f}")
        nc = max(int(out[27]), 1)
        lib.strait_replay_cta_profile(cw.ctypes.data)
        if out[27]:
            w = cw.reshape(3, 16)[:, :8] / max(int(out[27]), 1)
            print("  CTA propose job, per warp (cycles after the post): wake " + " ".join(f"{v:.0f}" for v in w[0]) +
                  " | phase A end " + " ".join(f"{v:.0f}" for v in w[1]) + " | phase B end " +
                  " ".join(f"{v:.0f}" for v in w[2]))
            print(f"  CTA proposes {out[27]}: post..join {out[24] / nc:.0f} cyc (master wait at phase A end "
                  f"{out[25] / nc:.0f}), master combine {out[26] / nc:.0f} cyc; master phase A {out[28] / nc:.0f}, "
                  f"phase B {out[29] / nc:.0f}, join wait {out[30] / nc:.0f}")
        w = max(int(out[18]), 1)
        print(f"  per wide propose: mean kmax {out[21] / w:.2f}, no GPU with a slot {100 * out[22] / w:.1f}%, "
              f"running entries {out[23] / w:.2f}")


if __name__ == "__main__":
    main()
