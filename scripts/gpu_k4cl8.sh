# 8-CTA (2×2 pairs) multicast K4: bit-exactness first (bounded), then the K3+K4 loop with and without it.
timeout 240 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "k4_hybrid" 2>&1 | tail -2 || exit 1
for v in 0 1 0 1; do RF_K4_CL8=$v timeout 300 python scripts/k4_energy.py --gm 8 --reps 6 2>&1 | grep rand | sed "s/^/cl8=$v /"; done
