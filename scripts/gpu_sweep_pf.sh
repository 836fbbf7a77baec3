# sweep: L2 prefetch distance
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_bench_parity_gpu.py -q -x -p no:cacheprovider -k "sweep or c3 or round" 2>&1 | tail -1
for pf in 0 1 2 3 4; do
  STRAIT_SWEEP_PREFETCH=$pf timeout 300 python bench.py --steps 500 --warmup 5 --no-replay --no-single --e2e-steps 1 --no-cpu-baseline --no-parity 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('pf=$pf', round(r['kernel_ms'],4), round(d['ms_per_step'],4), round(r['frac_survey_basis'],3), d['clocks']['reasons'])"
done
