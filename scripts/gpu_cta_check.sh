# replay-engine iteration check: both layouts vs the goldens, single-replay speeds, phase profile
nvidia-smi -L
timeout 600 python -m pytest tests/test_replay_cta_gpu.py tests/test_replay_gpu.py tests/test_bench_parity_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1
timeout 600 python scripts/cta_probe.py 2000 20000 2>&1 | cut -c1-220
STRAIT_LIB=build/prof/_strait.so timeout 600 python scripts/replay_profile.py 3000 2.5 20000 > gpurun_out/replay_profile.txt 2>&1; grep "==\|TOTAL\|CTA prop" gpurun_out/replay_profile.txt
