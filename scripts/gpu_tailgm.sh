# Hybrid K4: raster group of the pair-cluster tail kernel (RF_TAIL_GM; 8 = default), interleaved, 8 launches each.
for g in 8 4 8 4 2; do RF_TAIL_GM=$g timeout 600 python scripts/k4_energy.py --gm 8 --reps 8 2>&1 | grep rand | sed "s/^/tail_gm=$g /"; done
