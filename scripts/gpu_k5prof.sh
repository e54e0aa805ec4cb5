set -x
mkdir -p gpurun_out
timeout 300 python scripts/k5_bench.py --n 131072 --p 512 > gpurun_out/k5.log 2>&1
timeout 300 python scripts/k5_bench.py --n 65536 --p 1024 >> gpurun_out/k5.log 2>&1
timeout 300 python scripts/k5_bench.py --n 131072 --p 512 --prec 3xtf32 >> gpurun_out/k5.log 2>&1
cat gpurun_out/k5.log
timeout 300 python scripts/k5_bench.py --n 32768 --p 512 --reps 1 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 1 -c 1 \
  -o gpurun_out/k5_full python scripts/k5_bench.py --n 32768 --p 512 --reps 1 > gpurun_out/ncu_k5.log 2>&1
tail -3 gpurun_out/ncu_k5.log
