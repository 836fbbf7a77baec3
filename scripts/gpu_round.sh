# Round check on the GPU box (run under gpurun): tests, smoke, bench lines of both arms,
# single-replay layouts, replay phase profile, ncu launch list + sweep capture (CSV only).
nvidia-smi -L
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -1 gpurun_out/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 1500 python bench.py > gpurun_out/bench.txt 2>&1; tail -1 gpurun_out/bench.txt | cut -c1-300
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.txt 2>&1; tail -1 gpurun_out/bench_ref.txt | cut -c1-200
timeout 900 python scripts/cta_probe.py 2000 20000 > gpurun_out/cta_probe.txt 2>&1; cut -c1-200 gpurun_out/cta_probe.txt
timeout 600 python scripts/propose_latency.py 2000 > gpurun_out/propose_latency.json 2>&1; tail -1 gpurun_out/propose_latency.json
STRAIT_LIB=build/prof/_strait.so timeout 600 python scripts/replay_profile.py 3000 2.5 20000 > gpurun_out/replay_profile.txt 2>&1
bash scripts/ncu_sweep2.sh
python scripts/ncu_traffic.py gpurun_out/raw_sweep.csv "ncu --set full, 1 launch of strait_round, cold cache, clocks unlocked (scripts/ncu_sweep2.sh)"
cp profiles/sweep_traffic.json gpurun_out/
