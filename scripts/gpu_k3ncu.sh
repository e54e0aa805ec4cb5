# Full ncu capture of K3's multicast kernel (the first tc_gemm launch of the 4th step of the bench command).
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-trf --no-phi4 --no-ridge"
timeout 300 $B > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc_gemm -s 15 -c 1 -o gpurun_out/k3mc_full -f $B > gpurun_out/ncu_k3mc.log 2>&1
tail -2 gpurun_out/ncu_k3mc.log
