for occ in 1 4; do
  STRAIT_REPLAY_OCC=$occ timeout 900 compute-sanitizer --tool racecheck --racecheck-report all python scripts/replay_one.py 3 150 > gpurun_out/san_rc_$occ.txt 2>&1
  grep -E "RACECHECK SUMMARY" gpurun_out/san_rc_$occ.txt
done
grep -m 8 -E "Warning|Error" gpurun_out/san_rc_1.txt
