"""Where the C4 end-to-end step goes beyond the device launch: host batch
build (configs, stream descriptions, H2D, device stream generation), the
replay + metrics launch, and result() (D2H of the fetched outputs), each timed
alone, then the pipelined loop at 4 and 8 steps.

    python scripts/c4_e2e_probe.py
"""
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    import torch

    from paper_2604_28175_b200.configs import c4_grid
    from paper_2604_28175_b200.replay import ReplayBatch, ReplaySpec
    from paper_2604_28175_b200.shard import lpt

    sys.path.insert(0, REPO)
    from bench import expected_requests

    grid = c4_grid()
    specs = [ReplaySpec(*grid[i]) for i in lpt([expected_requests(c) for c, _ in grid], 1)[0]]
    fetch = {"counters", "req_status", "req_violated"}
    out = {}

    def timed(fn):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        return r, (time.perf_counter() - t0) * 1e3

    b, _ = timed(lambda: ReplayBatch(specs, generate="device"))
    b, out["build_ms"] = timed(lambda: ReplayBatch(specs, generate="device"))
    p, out["launch_ms"] = timed(lambda: b.launch(metrics=True))
    _, out["result_ms"] = timed(lambda: p.result(fetch=fetch))
    p, out["launch_nometrics_ms"] = timed(lambda: b.launch(metrics=False))
    p.result(fetch=fetch)
    s_build, s_run = torch.cuda.Stream(), torch.cuda.Stream()

    def build():
        with torch.cuda.stream(s_build):
            return ReplayBatch(specs, generate="device")

    for n in (4, 8):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        nxt = build()
        for i in range(n):
            cur = nxt
            s_run.wait_stream(s_build)
            pend = cur.launch(stream=s_run, metrics=True)
            nxt = build() if i + 1 < n else None
            pend.result(fetch=fetch)
        torch.cuda.synchronize()
        out[f"pipelined_{n}_ms_per_step"] = (time.perf_counter() - t0) * 1e3 / n
    out["requests"] = int(b.N)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
