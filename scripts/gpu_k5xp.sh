for gm in 1 4 64; do for b in 0 1; do RF_GM5=$gm RF_K5_BLOCKED=$b timeout 300 python scripts/k5_bench.py --n 131072 --p 512 2>&1 | sed "s/^/gm=$gm blocked=$b /"; done; done
