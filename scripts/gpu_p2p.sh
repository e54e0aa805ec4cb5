mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_p2p.py -q -s > gpurun_out/pytest_p2p.log 2>&1; grep -E "parity|passed|failed|^E |Error" gpurun_out/pytest_p2p.log | head -30
