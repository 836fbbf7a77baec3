# object-API node runtime on the GPU: node tests, scheduler tests, propose latency
nvidia-smi -L
timeout 900 python -m pytest tests/test_node_gpu.py tests/test_scheduler_gpu.py tests/test_acceptance_criteria_gpu.py tests/test_predictor_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_node.txt 2>&1; tail -15 gpurun_out/pytest_node.txt
timeout 300 python scripts/propose_latency.py 2000 > gpurun_out/propose_latency.json 2>&1; cat gpurun_out/propose_latency.json | tail -3
