# K3^ter multicast hybrid: parity, then the TRF timing (K3^ter, K4^ter) with and without it.
timeout 600 python -m pytest tests/test_gpu_trf.py -m gpu -q -x 2>&1 | tail -2
for v in 0 1 0 1; do echo -n "RF_K3_MC=$v: "; RF_K3_MC=$v timeout 600 python scripts/trf_bench.py --eps 0.9 --reps 6 2>&1 | grep TRF; done
