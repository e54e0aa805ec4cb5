# Soft-lockstep parameter sweep on the hybrid K4 (RF_LOCKW lead in K-blocks, RF_LOCKKS check period), interleaved.
for v in "RF_LOCKW=24 RF_LOCKKS=8" "RF_LOCKW=16 RF_LOCKKS=8" "RF_LOCKW=40 RF_LOCKKS=8" "RF_LOCKW=24 RF_LOCKKS=4" "RF_LOCKW=24 RF_LOCKKS=8" "RF_LOCKW=64 RF_LOCKKS=16"; do
  env $v timeout 300 python scripts/k4_energy.py --gm 8 --reps 6 2>&1 | grep rand | sed "s/^/$v /"; done
