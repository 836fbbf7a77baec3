# ncu of the C3 sweep kernel (strait_round): launch list + one --set full capture; CSV exports only
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-replay --no-single --no-parity > /tmp/ncu_launch_run.txt 2>&1
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:sweep_ws -s 3 -c 1 -o /tmp/prof_sweep python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-replay --no-single --no-parity > /tmp/ncu_full_run.txt 2>&1
ncu -i /tmp/prof_sweep.ncu-rep --page raw --csv > gpurun_out/raw_sweep.csv 2>/dev/null
ncu -i /tmp/prof_sweep.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_sweep.csv 2>/dev/null
# (the .ncu-rep itself stays on the box: gpurun_out/ is capped at 64 MiB)
tail -2 /tmp/ncu_full_run.txt
python scripts/ncu_summary.py gpurun_out/raw_sweep.csv
