# sweep pipeline shape: stages x consumer groups
for ns in 2 3 4; do for gr in 1 2; do
  STRAIT_SWEEP_STAGES=$ns STRAIT_SWEEP_GROUPS=$gr timeout 300 python bench.py --steps 200 --warmup 3 --e2e-steps 2 --no-cpu-baseline --no-replay 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ns=$ns gr=$gr', round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],3), d['checksum'])"
done; done
