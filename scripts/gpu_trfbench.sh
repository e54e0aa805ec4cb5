mkdir -p gpurun_out
for e in 0.9 0.0; do timeout 300 python scripts/trf_bench.py --eps $e 2>&1 | tail -2; done
