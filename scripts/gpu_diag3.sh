# needs a diagnostics build: make clean-free rebuild of strait_sweep.o with -DSTRAIT_SWEEP_DIAG_BUILD=1
# certified fast projections vs exact-only (diag 32)
for diag in 0 32; do
  STRAIT_SWEEP_DIAG=$diag timeout 300 python bench.py --steps 50 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-replay 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('diag=$diag', round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],3), d['checksum'] if 'checksum' in d else '')"
done
