# K3 raster group sweep (RF_GM3) inside the K3+K4 loop of scripts/k4_energy.py, interleaved.
for g in 8 4 16 32 8 4 16 32; do RF_GM3=$g timeout 600 python scripts/k4_energy.py --gm 8 --reps 6 2>&1 | grep rand | sed "s/^/gm3=$g /"; done
