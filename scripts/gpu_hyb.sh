timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1
RF_DEBUG_LAUNCH=1 timeout 180 python scripts/check_hybrid.py 2>&1 | grep -E "exact|DIFF"
timeout 300 python scripts/k4_energy.py --gm 8 --reps 2 2>&1 | grep rand
timeout 300 python scripts/trf_bench.py --eps 0.9 2>&1 | grep TRF
