# Full ncu capture (with source) of K5 at configs[4] shape.
mkdir -p gpurun_out
timeout 300 python scripts/k5_bench.py --reps 1 2>&1 | tail -1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc_gemm -s 1 -c 1 -o gpurun_out/k5_c4_full -f \
  python scripts/k5_bench.py --reps 1 > gpurun_out/ncu_k5_c4.log 2>&1; tail -3 gpurun_out/ncu_k5_c4.log
