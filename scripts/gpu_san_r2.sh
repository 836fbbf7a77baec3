# round-2 sanitizers: the CTA-per-replay engine and the sweep's 1- and 3-group pipelines
nvidia-smi -L
for g in 1 3; do
  STRAIT_SWEEP_GROUPS=$g STRAIT_SWEEP_STAGES=4 timeout 120 python bench.py --steps 3 --warmup 3 --segments 4096 --no-replay --no-single --e2e-steps 1 --no-cpu-baseline --no-parity > gpurun_out/g$g.txt 2>&1; echo "groups=$g rc=$?"
done
for tool in racecheck synccheck; do
  STRAIT_SWEEP_GROUPS=3 STRAIT_SWEEP_STAGES=4 timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_sweep3_$tool.txt 2>&1; echo "sweep groups=3 $tool rc=$?"
  timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_sweep1_$tool.txt 2>&1; echo "sweep groups=1 $tool rc=$?"
  STRAIT_REPLAY_NW=8 timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/replay_one.py 2 150 > gpurun_out/san_cta_$tool.txt 2>&1; echo "replay CTA $tool rc=$?"
done
STRAIT_REPLAY_NW=8 timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/replay_one.py 2 150 > gpurun_out/san_cta_memcheck.txt 2>&1; echo "replay CTA memcheck rc=$?"
tail -2 gpurun_out/san_*.txt
