# Round evidence on one B200 (call 1 of 2): tests, smoke, bench line, reference arm, then the launch list of the
# bench command under ncu (gpu__time_duration + DRAM bytes per launch) after the same command exited 0 without ncu.
# Call 2 (scripts/gpu_k5ncu4.sh / a K4 capture) takes the one `ncu --set full` capture.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1; tail -1 gpurun_out/bench_ref.json
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-trf --no-phi4 --no-ridge"
timeout 300 $B > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1
ls -la gpurun_out
