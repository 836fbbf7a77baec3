import sys; sys.path[:0]=['/root/repo','/root/repo/tests']
import numpy as np, torch
import test_scheduler_gpu as T
from paper_2604_28175_b200 import scheduler as S, sweep as SW, _device as D
from oracle import oracle
pred = T.one_metric_predictor()
gpu = T.mk_gpu()
run_p = T.mk_profile("hp-run", deadline_ms=100.0, base_total=16.0, transfer_frac=0.25, kernel_frac=0.5, throughput_row=(0.0,), self_compute=0.0, self_memory=0.0)
e = T.running(gpu, run_p, 1, now=4.0, kernel_start=0.0, deadline_abs=12.0)
cand = T.mk_profile("hp-cand", deadline_ms=500.0, throughput_row=(1.0,), self_compute=0.0, self_memory=0.0)
soa, agg = S._snapshot(cand, [1], 0.0, [gpu], 4.0, pred)
host = {k: D.host(v) for k, v in soa.arrays.items()}
print("twa dev", host["ent_twa"])
P = np.array(pred.params.to_vector())
print("P", P)
for C in (1, 2, 4):
    h = dict(host)
    for k in [k for k in h if k.startswith("ent_")]:
        a = h[k]
        if a.ndim == 2:
            b = np.zeros((a.shape[0], C), a.dtype); b[:, :1] = a
        else:
            b = np.zeros(C, a.dtype); b[:1] = a
            if k == "ent_t_kernel": b[1:] = 1.0
        h[k] = b
    hs = soa.like(h); hs.n_slots = C
    dev = SW.sweep(hs, P)
    orc = oracle.sweep(hs, P)
    print("C", C, "dev", dev["pair_flags"], dev["seg_gpu"], dev["seg_latency"], "oracle", orc["pair_flags"], orc["seg_gpu"])
# direct predict of the projection inputs
from paper_2604_28175_b200.predictor import predict_parts_batch
print(predict_parts_batch(pred.params, [[1.0]], 0.0, 0.0, 0))
print(predict_parts_batch(pred.params, [[0.0]], 0.0, 0.0, 0))
