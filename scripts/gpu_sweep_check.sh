# sweep iteration check: parity tests, timing, sanitizers on the smoke sweep
nvidia-smi -L
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_bench_parity_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1
for i in 1 2; do
  timeout 300 python bench.py --steps 500 --warmup 5 --no-replay --no-single --e2e-steps 1 --no-cpu-baseline --no-parity 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('kernel_ms', round(r['kernel_ms'],4), 'frac', round(r['frac'],3), d['clocks']['reasons'], d['clocks']['sm_mhz'])"
done
for tool in racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_sweep_$tool.txt 2>&1; echo "sweep $tool rc=$?"
done
STRAIT_SWEEP_GROUPS=2 STRAIT_SWEEP_STAGES=2 timeout 300 python bench.py --steps 100 --warmup 3 --no-replay --no-single --e2e-steps 1 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('groups=2', round(d['roofline']['kernel_ms'],4), d['parity'])"
