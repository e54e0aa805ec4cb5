set -x
mkdir -p gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,lts__throughput.avg.pct_of_peak_sustained_elapsed"
timeout 300 python scripts/k4_energy.py --gm 8 --reps 1 > gpurun_out/plain.log 2>&1 && \
for gm in 1 8 16 32; do
  RF_GM=$gm timeout 600 ncu --metrics $M --clock-control none -k regex:tc_gemm -s 1 -c 1 --csv \
    --log-file gpurun_out/k4m_gm$gm.csv python scripts/k4_energy.py --gm $gm --reps 1 > gpurun_out/ncu_gm$gm.log 2>&1
done
ls gpurun_out
