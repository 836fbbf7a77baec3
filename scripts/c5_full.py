"""BASELINE configs[4] at full size: the whole ~100M-request C5 replay (64
simulated GPUs, 20 models, bursty HP trace, 1,923 s) on one B200, timed on
the device with its streams drawn on the device, then the CPU oracle on the
same replay (host numpy streams, one core) and a comparison of every
per-request, per-decision, per-batch and cap-row array and the counters.

    python scripts/c5_full.py [--no-oracle]      -> one JSON line
"""
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    import torch

    from bench import REPLAY_COMPARE, COUNTER_COMPARE, time_launches
    from paper_2604_28175_b200.configs import C5_DURATION_MS, c5_prefix
    from paper_2604_28175_b200.replay import RC, ReplayBatch, ReplaySpec

    cfg = c5_prefix(duration=C5_DURATION_MS)
    spec = ReplaySpec(cfg, cfg.seed)
    t0 = time.perf_counter()
    batch = ReplayBatch([spec], generate="device")
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    dev_ms, launches, counters = time_launches(batch, 1, warm=0)
    c = counters[0]
    out = {"workload": "C5 full (BASELINE configs[4]): 64 GPUs, 20 models, bursty HP trace, 1,923 s",
           "requests": int(batch.N), "device_s": dev_ms / 1e3, "value": batch.N / (dev_ms / 1e3),
           "unit": "simulated requests/s", "input_build_s": build_s, "gpu_launches": launches,
           "batches": int(c[RC["BATCHES"]]), "passes": int(c[RC["PASSES"]]),
           "hp_violation_pct": 100.0 * c[RC["HP_VIOL"]] / max(c[RC["HP_ARR"]], 1),
           "lp_violation_pct": 100.0 * c[RC["LP_VIOL"]] / max(c[RC["LP_ARR"]], 1)}
    print(json.dumps(out), flush=True)
    if "--no-oracle" in sys.argv:
        return
    from oracle import oracle

    t0 = time.perf_counter()
    res = ReplayBatch([spec], generate="device").run(metrics=False)
    torch.cuda.synchronize()
    out["e2e_run_s"] = time.perf_counter() - t0
    host = ReplayBatch([spec])
    t0 = time.perf_counter()
    ref = oracle.replay(host, threads=1)
    out["oracle_1core_s"] = time.perf_counter() - t0
    a, b = ref.replay_slice(0), res.replay_slice(0)
    bad = []
    for k in REPLAY_COMPARE:
        x, y = np.asarray(a[k]), np.asarray(b[k])
        if k == "counters":
            x, y = x[..., COUNTER_COMPARE], y[..., COUNTER_COMPARE]
        if x.shape != y.shape or not np.array_equal(x, y, equal_nan=x.dtype.kind == "f"):
            bad.append(k)
    out["parity"] = {"ok": not bad, "arrays": len(REPLAY_COMPARE), "mismatches": bad, "requests": int(host.N)}
    out["cpu_baseline"] = {"value": host.N / out["oracle_1core_s"], "unit": "simulated requests/s", "cores": 1,
                           "kind": "port", "sample": "the whole replay on 1 core (oracle/strait_replay_oracle.c)"}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
