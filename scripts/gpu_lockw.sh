# Soft-lockstep window (K-blocks of lead) on the hybrid K4, via k4_energy.py --lockw, interleaved.
for i in 1 2; do for w in 24 12 40 24 64; do
  timeout 300 python scripts/k4_energy.py --gm 8 --reps 6 --lockw $w 2>&1 | grep rand | cut -c1-100; done; done
