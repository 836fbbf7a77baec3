# sweep pipeline shape after the LP-cap short-circuit: stages x consumer groups
for ns in 2 3 4; do for gr in 1 2; do
  STRAIT_SWEEP_STAGES=$ns STRAIT_SWEEP_GROUPS=$gr timeout 300 python bench.py --steps 300 --warmup 3 --no-replay --no-single --e2e-steps 1 --no-cpu-baseline --no-parity 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('ns=$ns gr=$gr', round(r['kernel_ms'],4), round(r['frac'],3), d['clocks']['reasons'])"
done; done
