# needs a diagnostics build: make clean-free rebuild of strait_sweep.o with -DSTRAIT_SWEEP_DIAG_BUILD=1
# sweep compute split: full, compute-only (4), no projections (8), both (12), no meet predict (16)
for diag in 0 4 8 12 16 2; do
  STRAIT_SWEEP_DIAG=$diag timeout 300 python bench.py --steps 30 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-replay 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('diag=$diag', round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],3))"
done
