mkdir -p gpurun_out
for e in 0 10; do RF_EXP_EPI=$e timeout 300 python scripts/k5_bench.py --n 131072 --p 512 2>&1 | sed "s/^/exp=$e /"; done
for e in 0 10; do RF_EXP_EPI=$e timeout 300 python scripts/k5_bench.py --n 65536 --p 1024 2>&1 | sed "s/^/exp=$e /"; done
