set -x
mkdir -p gpurun_out
timeout 600 python scripts/k4_energy.py --gm 1,4,8,16,32 --zero > gpurun_out/k4_energy.log 2>&1
cat gpurun_out/k4_energy.log
timeout 300 python scripts/k4_energy.py --gm 8 --reps 1 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:EpiSyrk -s 1 -c 1 \
  -o gpurun_out/k4_full python scripts/k4_energy.py --gm 8 --reps 1 > gpurun_out/ncu_k4.log 2>&1
tail -3 gpurun_out/ncu_k4.log
