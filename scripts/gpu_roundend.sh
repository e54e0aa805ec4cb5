#!/bin/bash
# Round-end evidence on one B200: GPU suite, smoke, default bench, ncu launch list (time + DRAM bytes) of one step.
# Usage (from the repo root, under gpurun): bash scripts/gpu_roundend.sh <tag>
tag=${1:-re}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $out/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "rc=$?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "rc=$?" >> $out/smoke.log
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "rc=$?" >> $out/bench.err
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    --csv --log-file $out/traffic.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-trf --no-phi4 \
    --no-cpu-baseline > $out/ncu.log 2>&1; echo "rc=$?" >> $out/ncu.log
