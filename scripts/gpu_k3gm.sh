mkdir -p gpurun_out
for gm in 8 32 64 256; do RF_GM3=$gm timeout 300 python scripts/k4_energy.py --gm 8 --reps 2 2>&1 | grep rand | sed "s/^/gm3=$gm /"; done
