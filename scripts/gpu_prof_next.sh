mkdir -p gpurun_out
timeout 300 python scripts/trf_bench.py --eps 0.9 --reps 1 > gpurun_out/plain_trf.log 2>&1 && cat gpurun_out/plain_trf.log && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 3 -c 1 -o gpurun_out/k4ter_full python scripts/trf_bench.py --eps 0.9 --reps 1 > gpurun_out/ncu_k4ter.log 2>&1
tail -2 gpurun_out/ncu_k4ter.log
