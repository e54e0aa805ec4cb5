# Hybrid multicast K3 (default): parity first (bounded), then the K3+K4 loop and the bench step.
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_acts.py tests/test_gpu_packed.py -m gpu -q -x 2>&1 | tail -2 || exit 1
for v in 0 1 0 1; do RF_K3_MC=$v timeout 600 python scripts/k4_energy.py --gm 8 --reps 6 2>&1 | grep rand | sed "s/^/k3mc=$v /"; done
for r in 110 120 135; do RF_HYB3_R100=$r timeout 600 python scripts/k4_energy.py --gm 8 --reps 6 2>&1 | grep rand | sed "s/^/r100=$r /"; done
