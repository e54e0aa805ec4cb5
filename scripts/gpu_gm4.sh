# Multicast K4 raster group (RF_GM4, super rows per group), interleaved.
for i in 1 2; do for g in 8 12 16 4; do RF_GM4=$g timeout 300 python scripts/k4_energy.py --gm 8 --reps 6 2>&1 | grep rand | sed "s/^/gm4=$g /" | cut -c1-100; done; done
