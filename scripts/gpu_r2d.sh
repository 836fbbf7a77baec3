# round-2 bench lines (ours + reference arm) and the sweep ncu capture
nvidia-smi -L
timeout 1500 python bench.py > gpurun_out/bench.txt 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench.txt | cut -c1-300
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.txt 2>&1; echo ref rc=$?; tail -1 gpurun_out/bench_ref.txt | cut -c1-300
bash scripts/ncu_sweep2.sh
