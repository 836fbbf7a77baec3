# quick bench shake-out on the GPU box (ours only; short C3 leg)
nvidia-smi -L
timeout 1500 python bench.py --steps 50 --warmup 3 > gpurun_out/bench_quick.txt 2>&1; echo rc=$?
tail -1 gpurun_out/bench_quick.txt | cut -c1-600
