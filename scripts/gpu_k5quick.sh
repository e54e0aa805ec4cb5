set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python scripts/k5_bench.py --n 131072 --p 512 > gpurun_out/k5.log 2>&1
timeout 300 python scripts/k5_bench.py --n 65536 --p 1024 >> gpurun_out/k5.log 2>&1
timeout 300 python scripts/k5_bench.py --n 131072 --p 512 --prec 3xtf32 >> gpurun_out/k5.log 2>&1
timeout 300 python scripts/k4_energy.py --gm 8 --reps 2 >> gpurun_out/k5.log 2>&1
cat gpurun_out/k5.log
