for gm in 16 32 64 128 512; do RF_GM5=$gm timeout 300 python scripts/k5_bench.py --n 131072 --p 512 2>&1 | sed "s/^/gm5=$gm /"; done
for gm in 16 64; do RF_GM5=$gm timeout 300 python scripts/k5_bench.py --n 65536 --p 1024 2>&1 | sed "s/^/gm5=$gm /"; done
