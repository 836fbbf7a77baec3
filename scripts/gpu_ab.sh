# A/B of sweep builds: STRAIT_LIB variants
for lib in paper_2604_28175_b200/_strait.so build/v0/_strait.so build/v1/_strait.so; do for diag in 0 32; do
  STRAIT_LIB=$lib STRAIT_SWEEP_DIAG=$diag timeout 300 python bench.py --steps 50 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-replay 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib diag=$diag', round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],3))"
done; done
