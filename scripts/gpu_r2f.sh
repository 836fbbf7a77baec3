nvidia-smi -L
timeout 900 python -m pytest tests/test_replay_cta_gpu.py tests/test_replay_gpu.py tests/test_bench_parity_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_replay.txt 2>&1; tail -2 gpurun_out/pytest_replay.txt
timeout 900 python scripts/cta_probe.py 2000 20000 > gpurun_out/cta_probe.txt 2>&1; cat gpurun_out/cta_probe.txt | cut -c1-300
STRAIT_LIB=build/prof/_strait.so timeout 600 python scripts/replay_profile.py 3000 2.5 20000 > gpurun_out/replay_profile.txt 2>&1; grep "==\|TOTAL\|propose\|CTA" gpurun_out/replay_profile.txt
grep "CTA proposes" gpurun_out/replay_profile.txt
