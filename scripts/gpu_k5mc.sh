# K5 multicast hybrid: parity (bounded), then K5 at configs[4] / configs[3] shapes with and without it.
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_packed_tri.py tests/test_gpu_acts.py -m gpu -q -x 2>&1 | tail -2
for i in 1 2; do for v in 0 1; do
  echo -n "RF_K5_HYBRID=$v c4: "; RF_K5_HYBRID=$v timeout 300 python scripts/k5_bench.py --reps 5 2>&1 | tail -1
  echo -n "RF_K5_HYBRID=$v c3: "; RF_K5_HYBRID=$v timeout 300 python scripts/k5_bench.py --n 65536 --p 1024 --reps 5 2>&1 | tail -1
done; done
