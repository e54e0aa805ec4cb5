for h in 1 0 1 0; do RF_K4_HYBRID=$h timeout 600 python scripts/k4_energy.py --gm 8 --reps 8 2>&1 | grep rand | sed "s/^/hyb=$h /"; done
for h in 1 0; do RF_K4_HYBRID=$h timeout 600 python scripts/trf_bench.py --eps 0.9 --reps 10 2>&1 | grep TRF | sed "s/^/hyb=$h /"; done
