# ncu of the replay kernel at R replays (arg 1), OCC variant (arg 2); CSV exports only
R=${1:-2368}; OCC=${2:-4}
STRAIT_REPLAY_OCC=$OCC timeout 900 ncu --set full --clock-control none --import-source on -k regex:replay_kernel -c 1 -o /tmp/prof_replay python scripts/replay_one.py $R 1000 > /tmp/ncu_replay.txt 2>&1
tail -1 /tmp/ncu_replay.txt
ncu -i /tmp/prof_replay.ncu-rep --page raw --csv > gpurun_out/raw_replay_$R.csv 2>/dev/null
ncu -i /tmp/prof_replay.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_replay_$R.csv 2>/dev/null
