nvidia-smi -L
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 env STRAIT_REPLAY_NW=8 python scripts/replay_one.py 2 150 > gpurun_out/san_cta_synccheck.txt 2>&1; echo "replay CTA synccheck rc=$?"; tail -2 gpurun_out/san_cta_synccheck.txt
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 env STRAIT_REPLAY_NW=8 python scripts/replay_one.py 2 150 > gpurun_out/san_cta_racecheck.txt 2>&1; echo "replay CTA racecheck rc=$?"; tail -2 gpurun_out/san_cta_racecheck.txt
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_bench_parity_gpu.py tests/test_replay_cta_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_sweep.txt 2>&1; tail -2 gpurun_out/pytest_sweep.txt
timeout 1500 python bench.py > gpurun_out/bench.txt 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('kernel_ms', round(r['kernel_ms'],4), 'frac', round(r['frac'],3), d['parity'], d['clocks'], {k: round(d[k]['value']) for k in ('c1','c2','c4','c5')})"
bash scripts/ncu_sweep2.sh
python scripts/ncu_traffic.py gpurun_out/raw_sweep.csv "ncu --set full, 1 launch of strait_round, cold cache, clocks unlocked (scripts/ncu_sweep2.sh, round 2)"
cp profiles/sweep_traffic.json gpurun_out/
