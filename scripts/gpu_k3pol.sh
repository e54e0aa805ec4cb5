# K3 hybrid: evict_last operand loads (RF_K3_LOADPOL=1) vs normal, 5 interleaved pairs (K3 times from k4_energy.py).
for i in 1 2 3 4 5; do for v in 0 1; do
  RF_K3_LOADPOL=$v timeout 300 python scripts/k4_energy.py --gm 8 --reps 6 2>&1 | grep rand | sed "s/^/pol=$v /" | cut -c1-90; done; done
