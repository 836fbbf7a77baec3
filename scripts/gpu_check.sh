# GPU-box check: parity tests, smoke, bench config sweep, optional ncu.
#   bash scripts/gpu_check.sh [quick|full]
MODE=${1:-full}
nvidia-smi -L
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
timeout 600 python bench.py > gpurun_out/bench.txt 2>&1; tail -1 gpurun_out/bench.txt | cut -c1-400
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.txt 2>&1; tail -1 gpurun_out/bench_ref.txt | cut -c1-300
if [ "$MODE" = full ]; then
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_launch_run.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_ws -s 3 -c 1 -o gpurun_out/prof_sweep python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_full_run.txt 2>&1
fi
ls gpurun_out
