# A/B of K5 under an env switch (experiments), interleaved, at configs[4] and configs[3] shapes.
SW=${SW:-RF_K5_W12}
for i in 1 2; do
  for v in 0 1; do
    echo -n "$SW=$v c4: "; env $SW=$v timeout 300 python scripts/k5_bench.py --reps 5 2>&1 | tail -1
    echo -n "$SW=$v c3: "; env $SW=$v timeout 300 python scripts/k5_bench.py --n 65536 --p 1024 --reps 5 2>&1 | tail -1
  done
done
