# K3 hybrid split sweep (RF_HYB3_R100 = per-SM rate ratio ×100), interleaved.
for i in 1 2; do for r in 120 100 140 160; do RF_HYB3_R100=$r timeout 300 python scripts/k4_energy.py --gm 8 --reps 6 2>&1 | grep rand | sed "s/^/r100=$r /" | cut -c1-60; done; done
