set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_trf.py -x -q -s > gpurun_out/pytest_trf.log 2>&1; grep -E "parity|passed|failed|Error|assert" gpurun_out/pytest_trf.log | head -40
