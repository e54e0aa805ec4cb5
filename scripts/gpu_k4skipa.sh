# Experiment: K4 hybrid with the A-operand loads skipped (RF_EXP=1; wrong results, timing only): how much does
# L2 → SM traffic cost under the power cap?
for e in 0 1 0 1; do RF_EXP=$e timeout 300 python scripts/k4_energy.py --gm 8 --reps 6 2>&1 | grep rand | sed "s/^/exp=$e /"; done
