# ncu --set full of one C5-shape single replay (CTA layout), source-level CSV
cat > /tmp/c5one.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
from paper_2604_28175_b200.configs import c5
from paper_2604_28175_b200.replay import ReplayBatch, ReplaySpec
ReplayBatch([ReplaySpec(c5(300.0), 0)], generate="device").run(metrics=False)
PY
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:replay_kernel -c 1 -o /tmp/prof_c5 python /tmp/c5one.py > /tmp/ncu_c5.txt 2>&1
tail -1 /tmp/ncu_c5.txt
ncu -i /tmp/prof_c5.ncu-rep --page raw --csv > gpurun_out/raw_c5.csv 2>/dev/null
ncu -i /tmp/prof_c5.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_c5.csv 2>/dev/null
ls -la gpurun_out/src_c5.csv
