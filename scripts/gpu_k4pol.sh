# Hybrid K4 L2 policies (RF_K4_LOADPOL: 1 = evict_last operands; RF_K4_STOREPOL: 1 = evict_first G stores), interleaved.
for v in "RF_K4_LOADPOL=0 RF_K4_STOREPOL=0" "RF_K4_LOADPOL=1 RF_K4_STOREPOL=1" "RF_K4_LOADPOL=1 RF_K4_STOREPOL=0" "RF_K4_LOADPOL=0 RF_K4_STOREPOL=1" "RF_K4_LOADPOL=0 RF_K4_STOREPOL=0" "RF_K4_LOADPOL=1 RF_K4_STOREPOL=1" "RF_K4_LOADPOL=1 RF_K4_STOREPOL=0"; do
  env $v timeout 300 python scripts/k4_energy.py --gm 8 --reps 6 2>&1 | grep rand | sed "s/^/$v /" | cut -c1-130; done
