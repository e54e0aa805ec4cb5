set -x
mkdir -p gpurun_out
timeout 300 python scripts/k5_bench.py --n 65536 --p 512 --reps 1 > gpurun_out/plain.log 2>&1 && cat gpurun_out/plain.log && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 1 -c 1 \
  -o gpurun_out/k5_full2 python scripts/k5_bench.py --n 65536 --p 512 --reps 1 > gpurun_out/ncu_k5.log 2>&1
tail -3 gpurun_out/ncu_k5.log
