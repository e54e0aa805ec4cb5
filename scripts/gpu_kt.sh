# K̃ with 8 vs 12 epilogue warps (RF_KT_W12), parity with the default, centring post-pass rates.
timeout 600 python -m pytest tests -m gpu -q -x -k "ktilde or center" 2>&1 | tail -2
for v in 0 1 0 1; do echo "RF_KT_W12=$v"; RF_KT_W12=$v timeout 600 python scripts/center_bench.py 2>&1 | grep "K̃"; done
