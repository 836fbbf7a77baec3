"""CTA-per-replay engine (NW = 8 warps per replay) vs the one-warp engine
(STRAIT_REPLAY_NW=1) on single replays: every output array bit-identical
between the two, and each against the oracle; device time of each.

    python scripts/cta_probe.py [c5_ms] [c2_ms]   -> one JSON line per case
"""
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [REPO, os.path.join(REPO, "tests")]


def main():
    import torch

    from bench import COUNTER_COMPARE, REPLAY_COMPARE, time_launches
    from oracle import oracle
    from paper_2604_28175_b200.configs import c1, c5_prefix, overload
    from paper_2604_28175_b200.replay import ReplayBatch, ReplaySpec

    c5_ms = float(sys.argv[1]) if len(sys.argv) > 1 else 2000.0
    c2_ms = float(sys.argv[2]) if len(sys.argv) > 2 else 20000.0
    cases = [("c1", c1()), ("overload", overload(c2_ms)), ("c5", c5_prefix(duration=c5_ms))]
    for name, cfg in cases:
        spec = ReplaySpec(cfg, cfg.seed)
        out = {"case": name}
        res = {}
        for mode in ("1", "8"):
            os.environ["STRAIT_REPLAY_NW"] = mode
            b = ReplayBatch([spec], generate="device")
            dev_ms, _, _ = time_launches(b, 2, warm=1)
            res[mode] = ReplayBatch([spec], generate="device").run(metrics=False).replay_slice(0)
            out[f"nw{mode}_ms"] = dev_ms
            out["requests"] = int(b.N)
            out[f"nw{mode}_req_s"] = b.N / (dev_ms / 1e3)
        os.environ.pop("STRAIT_REPLAY_NW")
        host = ReplayBatch([spec])
        ref = oracle.replay(host, threads=1).replay_slice(0)
        bad = {"nw8_vs_nw1": [], "nw8_vs_oracle": []}
        for k in REPLAY_COMPARE:
            x, y, z = np.asarray(res["1"][k]), np.asarray(res["8"][k]), np.asarray(ref[k])
            if k == "counters":
                x, y, z = x[..., COUNTER_COMPARE], y[..., COUNTER_COMPARE], z[..., COUNTER_COMPARE]
            f = x.dtype.kind == "f"
            if x.shape != y.shape or not np.array_equal(x, y, equal_nan=f):
                bad["nw8_vs_nw1"].append(k)
            if z.shape != y.shape or not np.array_equal(z, y, equal_nan=f):
                bad["nw8_vs_oracle"].append(k)
        out["mismatches"] = bad
        out["ok"] = not bad["nw8_vs_nw1"] and not bad["nw8_vs_oracle"]
        out["speedup"] = out["nw1_ms"] / out["nw8_ms"]
        print(json.dumps(out), flush=True)
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
