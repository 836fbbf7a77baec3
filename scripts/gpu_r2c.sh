# round-2 check after the CTA engine + geometry + sweep-groups changes
nvidia-smi -L
timeout 900 python -m pytest tests/test_replay_gpu.py -q -x -p no:cacheprovider -k "geometry" > gpurun_out/pytest_geom.txt 2>&1; tail -3 gpurun_out/pytest_geom.txt
bash scripts/gpu_sweep_g3.sh
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 900 python scripts/cta_probe.py 2000 20000 > gpurun_out/cta_probe.txt 2>&1; cat gpurun_out/cta_probe.txt | cut -c1-300
STRAIT_LIB=build/prof/_strait.so timeout 600 python scripts/replay_profile.py 3000 2.5 20000 > gpurun_out/replay_profile.txt 2>&1; grep "==\|TOTAL\|arrival\|kernel_complete" gpurun_out/replay_profile.txt
