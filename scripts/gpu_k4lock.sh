set -x
mkdir -p gpurun_out
timeout 900 python scripts/k4_energy.py --gm 8,16,32 --lockw 0,8,24,64 --reps 2 > gpurun_out/k4_lock.log 2>&1
cat gpurun_out/k4_lock.log
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__cycles_elapsed.avg.per_second"
for lw in 8 24; do
  timeout 600 ncu --metrics $M --clock-control none -k regex:tc_gemm -s 1 -c 1 --csv \
    --log-file gpurun_out/k4m3_lw$lw.csv python scripts/k4_energy.py --gm 16 --lockw $lw --reps 1 > gpurun_out/ncu3_lw$lw.log 2>&1
done
