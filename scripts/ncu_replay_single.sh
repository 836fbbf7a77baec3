# ncu --set full of ONE single-replay launch (overload 3 s), source-level CSV; arg 1 = STRAIT_REPLAY_NW
NW=${1:-1}
STRAIT_REPLAY_NW=$NW timeout 900 ncu --set full --clock-control none --import-source on -k regex:replay_kernel -c 1 -o /tmp/prof_single_$NW python scripts/replay_one.py 1 3000 > /tmp/ncu_single.txt 2>&1
tail -1 /tmp/ncu_single.txt
ncu -i /tmp/prof_single_$NW.ncu-rep --page raw --csv > gpurun_out/raw_single_nw$NW.csv 2>/dev/null
ncu -i /tmp/prof_single_$NW.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_single_nw$NW.csv 2>/dev/null
ls -la gpurun_out/src_single_nw$NW.csv
