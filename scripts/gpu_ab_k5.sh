# A/B of K5 variants (env switches, experiments), interleaved, at configs[4] and configs[3] shapes.
for i in 1 2; do
  for v in "RF_K5_W12=0" "RF_K5_W12=1" "RF_K5_W16=1"; do
    echo -n "$v c4: "; env $v timeout 300 python scripts/k5_bench.py --reps 5 2>&1 | tail -1
    echo -n "$v c3: "; env $v timeout 300 python scripts/k5_bench.py --n 65536 --p 1024 --reps 5 2>&1 | tail -1
  done
done
RF_K5_W16=1 timeout 600 python -m pytest tests -m gpu -q -x -k "phi or Phi or eq1 or packed_tri" 2>&1 | tail -1
