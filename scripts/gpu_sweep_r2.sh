# sweep kernel A/B after the cap-skip multiply + pair work before the barrier; parity tests
nvidia-smi -L
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_bench_parity_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_sweep.txt 2>&1; tail -2 gpurun_out/pytest_sweep.txt
for cfg in "2 1" "4 3" "2 1" "4 3"; do set -- $cfg
  STRAIT_SWEEP_STAGES=$1 STRAIT_SWEEP_GROUPS=$2 timeout 300 python bench.py --steps 500 --warmup 5 --no-replay --no-single --e2e-steps 1 --no-cpu-baseline --no-parity 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('ns=$1 gr=$2', round(r['kernel_ms'],4), round(r['frac'],3), d['clocks']['reasons'], d['clocks']['sm_mhz'])"
done
