# K5 (16-warp, configs[4]) raster-group sweep (RF_GM5), interleaved.
for g in 16 32 64 8 16 32 64; do echo -n "gm5=$g: "; RF_GM5=$g timeout 300 python scripts/k5_bench.py --reps 5 2>&1 | tail -1 | cut -c1-90; done
