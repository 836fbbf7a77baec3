# Round check on the GPU box: tests, smoke, bench (ours + reference), ncu launch list + full captures (CSV only)
nvidia-smi -L
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -1 gpurun_out/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench.txt 2>&1; tail -1 gpurun_out/bench.txt | cut -c1-300
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.txt 2>&1; tail -1 gpurun_out/bench_ref.txt | cut -c1-200
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-replay > /tmp/ncu_launch_run.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_ws -s 3 -c 1 -o /tmp/prof_sweep python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-replay > /tmp/ncu_full_run.txt 2>&1
ncu -i /tmp/prof_sweep.ncu-rep --page raw --csv > gpurun_out/raw_sweep.csv 2>/dev/null
ncu -i /tmp/prof_sweep.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_sweep.csv 2>/dev/null
STRAIT_REPLAY_OCC=4 timeout 900 ncu --set full --clock-control none --import-source on -k regex:replay_kernel -c 1 -o /tmp/prof_replay python scripts/replay_one.py 1184 1000 > /tmp/ncu_replay.txt 2>&1
ncu -i /tmp/prof_replay.ncu-rep --page raw --csv > gpurun_out/raw_replay.csv 2>/dev/null
ncu -i /tmp/prof_replay.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_replay.csv 2>/dev/null
ls gpurun_out
