# sweep kernel: parity tests + short C3-only bench
nvidia-smi -L
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_bench_parity_gpu.py -q -x -p no:cacheprovider -k "sweep or c3 or round" > gpurun_out/pytest_sweep.txt 2>&1; tail -3 gpurun_out/pytest_sweep.txt
for i in 1 2; do
timeout 600 python bench.py --steps 500 --warmup 5 --no-replay --no-single --e2e-steps 2 --no-cpu-baseline > gpurun_out/bench_sweep.txt 2>&1
tail -1 gpurun_out/bench_sweep.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('kernel_ms', round(r['kernel_ms'],4), 'ms/step', round(d['ms_per_step'],4), 'frac', round(r['frac'],3), 'record', round(r['record_basis']['frac'],3), d['parity'], d['clocks'])"
done
