# CTA-per-replay engine iteration: parity + speed probe, phase profile, reference binding
nvidia-smi -L
timeout 900 python scripts/cta_probe.py 2000 20000 > gpurun_out/cta_probe.txt 2>&1; echo probe rc=$?; cat gpurun_out/cta_probe.txt | cut -c1-600
STRAIT_LIB=build/prof/_strait.so timeout 600 python scripts/replay_profile.py 3000 2.5 20000 > gpurun_out/replay_profile.txt 2>&1; cat gpurun_out/replay_profile.txt
STRAIT_REPLAY_NW=1 STRAIT_LIB=build/prof/_strait.so timeout 600 python scripts/replay_profile.py 3000 2.5 20000 > gpurun_out/replay_profile_nw1.txt 2>&1; grep "==\|TOTAL" gpurun_out/replay_profile_nw1.txt
timeout 600 python scripts/reference_binding.py 800 > gpurun_out/reference_binding.json 2>&1; tail -3 gpurun_out/reference_binding.json
