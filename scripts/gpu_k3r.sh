# K3 hybrid split sweep (RF_HYB3_R100 = per-SM rate ratio ×100), interleaved.
for r in 120 135 150 135 120 150; do RF_HYB3_R100=$r timeout 600 python scripts/k4_energy.py --gm 8 --reps 6 2>&1 | grep rand | sed "s/^/r100=$r /"; done
