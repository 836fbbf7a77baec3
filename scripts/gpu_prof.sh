# one ncu --set full capture of the sweep kernel + launch list
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_launch_run.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_ws -s 3 -c 1 -o gpurun_out/prof_sweep python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_full_run.txt 2>&1
tail -2 gpurun_out/ncu_full_run.txt
