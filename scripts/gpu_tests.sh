set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -s > gpurun_out/pytest_gpu.log 2>&1; grep -E "parity\] packed|passed|failed|Error|error" gpurun_out/pytest_gpu.log | tail -30
