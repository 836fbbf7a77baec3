# CTA-per-replay engine: parity + speed probe, GPU tests, phase profile, reference binding
nvidia-smi -L
timeout 900 python scripts/cta_probe.py 2000 20000 > gpurun_out/cta_probe.txt 2>&1; echo probe rc=$?; cat gpurun_out/cta_probe.txt | cut -c1-600
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -4 gpurun_out/pytest_gpu.txt
STRAIT_LIB=build/prof/_strait.so timeout 600 python scripts/replay_profile.py 3000 2.5 20000 > gpurun_out/replay_profile.txt 2>&1; cat gpurun_out/replay_profile.txt
timeout 600 python scripts/reference_binding.py 800 > gpurun_out/reference_binding.json 2>&1; tail -3 gpurun_out/reference_binding.json
