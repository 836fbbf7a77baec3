# needs a diagnostics build: make clean-free rebuild of strait_sweep.o with -DSTRAIT_SWEEP_DIAG_BUILD=1
# sweep kernel diagnostics: tensor-map vs bulk, data-movement-only vs full, stages/groups
nvidia-smi -L
python -m pytest tests -m gpu -q -p no:cacheprovider -k "sweep or round" > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
for path in 0; do for diag in 0 2; do for ns in 2 3 4; do for gr in 1 2; do
  STRAIT_SWEEP_PATH=$path STRAIT_SWEEP_DIAG=$diag STRAIT_SWEEP_STAGES=$ns STRAIT_SWEEP_GROUPS=$gr timeout 300 python bench.py --steps 30 --warmup 3 --e2e-steps 1 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('path=$path diag=$diag ns=$ns gr=$gr', round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],3), d['roofline']['kernel'])"
done; done; done; done
