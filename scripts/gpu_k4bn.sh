for b in 0 1 0 1; do RF_K4_BN256=$b timeout 300 python scripts/k4_energy.py --gm 8 --reps 2 2>&1 | grep rand | sed "s/^/bn256=$b /"; done
