# round-2 check after the CTA engine + geometry + sweep-groups changes
nvidia-smi -L
timeout 900 python -m pytest tests/test_replay_gpu.py -q -x -p no:cacheprovider -k "geometry" > gpurun_out/pytest_geom.txt 2>&1; tail -3 gpurun_out/pytest_geom.txt
bash scripts/gpu_sweep_g3.sh
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
