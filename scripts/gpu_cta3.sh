nvidia-smi -L
STRAIT_LIB=build/prof/_strait.so timeout 600 python scripts/replay_profile.py 3000 2.5 20000 > gpurun_out/replay_profile.txt 2>&1; cat gpurun_out/replay_profile.txt
bash scripts/ncu_replay_single.sh 1
bash scripts/ncu_replay_single.sh 8
