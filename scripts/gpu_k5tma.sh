# A/B: K5 Φ stores through smem + TMA (RF_K5_TMA=1, default) vs direct per-lane 128-B row stores (RF_K5_TMA=0),
# interleaved, at configs[4] and configs[3] shapes; then the Φ parity tests with direct stores.
for i in 1 2; do
  for v in 1 0; do
    echo -n "tma=$v c4: "; RF_K5_TMA=$v timeout 300 python scripts/k5_bench.py --reps 5 2>&1 | tail -1 | cut -c1-110
    echo -n "tma=$v c3: "; RF_K5_TMA=$v timeout 300 python scripts/k5_bench.py --n 65536 --p 1024 --reps 5 2>&1 | tail -1 | cut -c1-110
  done
done
RF_K5_TMA=0 timeout 600 python -m pytest tests -m gpu -q -x -k "phi or Phi or eq1 or packed_tri" 2>&1 | tail -1
