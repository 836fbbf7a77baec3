# ncu captures of the replay engine: 1 replay (latency) and 1184 replays (throughput)
nproc; lscpu | grep -E "Model name|Socket|Core|Thread" | head -5
timeout 600 ncu --set full --clock-control none --import-source on -k regex:replay_kernel -c 1 -o gpurun_out/prof_replay1 python scripts/replay_one.py 1 1000 > gpurun_out/ncu_replay1.txt 2>&1
tail -2 gpurun_out/ncu_replay1.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:replay_kernel -c 1 -o gpurun_out/prof_replay1184 python scripts/replay_one.py 1184 1000 > gpurun_out/ncu_replay1184.txt 2>&1
tail -2 gpurun_out/ncu_replay1184.txt
ls -la gpurun_out
