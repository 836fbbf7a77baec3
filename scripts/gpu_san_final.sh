# final sanitizer pass: CTA-layout replays (C5 geometry and forced on overload), one-warp replays, the sweep smoke
nvidia-smi -L
cat > /tmp/c5small.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
from paper_2604_28175_b200.configs import c5
from paper_2604_28175_b200.replay import ReplayBatch, ReplaySpec
r = ReplayBatch([ReplaySpec(c5(30.0), 0)]).run(metrics=False); r.check(); print("c5 ok")
PY
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python /tmp/c5small.py > gpurun_out/san_c5_$tool.txt 2>&1; echo "CTA c5 $tool rc=$?"
  STRAIT_REPLAY_NW=8 timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/replay_one.py 2 150 > gpurun_out/san_cta_$tool.txt 2>&1; echo "CTA overload $tool rc=$?"
  STRAIT_REPLAY_NW=1 timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/replay_one.py 2 150 > gpurun_out/san_nw1_$tool.txt 2>&1; echo "one-warp overload $tool rc=$?"
done
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_smoke_$tool.txt 2>&1; echo "smoke $tool rc=$?"
done
