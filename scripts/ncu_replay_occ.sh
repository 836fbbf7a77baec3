# ncu of the replay kernel at 2368 replays, both occupancy variants; CSV summaries only
for o in 1 4; do
  STRAIT_REPLAY_OCC=$o timeout 600 ncu --set full --clock-control none --import-source on -k regex:replay_kernel -c 1 -o /tmp/prof_occ$o python scripts/replay_one.py 2368 1000 > /tmp/ncu_occ$o.txt 2>&1
  ncu -i /tmp/prof_occ$o.ncu-rep --page raw --csv > gpurun_out/raw_occ$o.csv 2>/dev/null
  ncu -i /tmp/prof_occ$o.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_occ$o.csv 2>/dev/null
done
for o in 1 4; do STRAIT_REPLAY_OCC=$o python scripts/replay_one.py 2368 1000 2>&1 | tail -1; done
ls -la gpurun_out
