mkdir -p gpurun_out
RF_EXP_EPI=7 timeout 300 python scripts/k5_bench.py --n 65536 --p 128 --reps 1 > gpurun_out/plain.log 2>&1 && \
RF_EXP_EPI=7 timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 1 -c 1 \
  -o gpurun_out/k5_exp7 python scripts/k5_bench.py --n 65536 --p 128 --reps 1 > gpurun_out/ncu_k5.log 2>&1
tail -2 gpurun_out/ncu_k5.log
