# sweep compute split on the diag build: full, data only (2), compute only (4), no projections (8), no meet predict (16)
for diag in 0 2 4 8 16 24; do
  STRAIT_LIB=build/diag/_strait.so STRAIT_SWEEP_DIAG=$diag STRAIT_SWEEP_PREFETCH=0 timeout 300 python bench.py --steps 300 --warmup 3 --no-replay --no-single --e2e-steps 1 --no-cpu-baseline --no-parity 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('diag=$diag', round(r['kernel_ms'],4), d['clocks']['reasons'])"
done
