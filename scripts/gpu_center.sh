mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_center.py -x -q -s > gpurun_out/pytest_center.log 2>&1; grep -E "parity|passed|failed|Error|^E " gpurun_out/pytest_center.log | head -30
