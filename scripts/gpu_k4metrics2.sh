set -x
mkdir -p gpurun_out
timeout 600 python scripts/k4_energy.py --gm 1,8,16,32 > gpurun_out/k4_energy2.log 2>&1
timeout 600 python scripts/k4_energy.py --gm 8,16 --pad-g >> gpurun_out/k4_energy2.log 2>&1
cat gpurun_out/k4_energy2.log
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__cycles_elapsed.avg.per_second,lts__throughput.avg.pct_of_peak_sustained_elapsed"
for gm in 8 16; do
  RF_GM=$gm timeout 600 ncu --metrics $M --clock-control none -k regex:tc_gemm -s 1 -c 1 --csv \
    --log-file gpurun_out/k4m2_gm$gm.csv python scripts/k4_energy.py --gm $gm --reps 1 > gpurun_out/ncu2_gm$gm.log 2>&1
done
