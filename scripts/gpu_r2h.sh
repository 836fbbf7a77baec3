nvidia-smi -L
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 1500 python bench.py > gpurun_out/bench.txt 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('kernel_ms', round(r['kernel_ms'],4), 'frac', round(r['frac'],3), r['traffic_matches_kernel'], d['parity'], d['clocks'], {k: round(d[k]['value']) for k in ('c1','c2','c4','c5')}, 'e2e', round(d['e2e']['value']/1e9,3))"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.txt 2>&1; echo ref rc=$?; tail -1 gpurun_out/bench_ref.txt | cut -c1-200
