set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python scripts/k4_energy.py --gm 8 --lockw 24 --reps 3 > gpurun_out/k3k4.log 2>&1; cat gpurun_out/k3k4.log
timeout 300 python scripts/k4_energy.py --gm 8 --reps 1 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 2 -c 1 \
  -o gpurun_out/k3_full python scripts/k4_energy.py --gm 8 --reps 1 > gpurun_out/ncu_k3.log 2>&1
tail -3 gpurun_out/ncu_k3.log
