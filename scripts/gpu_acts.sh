mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_acts.py -q -s > gpurun_out/pytest_acts.log 2>&1; grep -E "parity|passed|failed|^E " gpurun_out/pytest_acts.log | head -80
