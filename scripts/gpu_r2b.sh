# round-2 check: GPU tests, smoke, default bench, propose latency, replay phase profile
nvidia-smi -L
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -4 gpurun_out/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 1500 python bench.py > gpurun_out/bench.txt 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench.txt | cut -c1-300
timeout 300 python scripts/propose_latency.py 2000 > gpurun_out/propose_latency.json 2>&1; tail -1 gpurun_out/propose_latency.json
STRAIT_LIB=build/prof/_strait.so timeout 600 python scripts/replay_profile.py 3000 2.5 20000 > gpurun_out/replay_profile.txt 2>&1; cat gpurun_out/replay_profile.txt
