# compute-sanitizer over small launches of every kernel family (memcheck, racecheck, synccheck)
set -x
for tool in memcheck racecheck synccheck; do
  STRAIT_REPLAY_OCC=1 timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/replay_one.py 3 150 > gpurun_out/san_replay1_$tool.txt 2>&1; echo "replay(latency) $tool rc=$?"
  STRAIT_REPLAY_OCC=4 timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/replay_one.py 6 150 > gpurun_out/san_replay4_$tool.txt 2>&1; echo "replay(throughput) $tool rc=$?"
done
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_smoke_memcheck.txt 2>&1; echo "smoke memcheck rc=$?"
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_smoke_racecheck.txt 2>&1; echo "smoke racecheck rc=$?"
tail -3 gpurun_out/san_*.txt
