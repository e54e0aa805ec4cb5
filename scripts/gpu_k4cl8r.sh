# 8-CTA K4 hybrid: work split sweep (RF_HYB_R100) against the 4-CTA default, interleaved.
for v in "RF_K4_CL8=0" "RF_K4_CL8=1 RF_HYB_R100=130" "RF_K4_CL8=1 RF_HYB_R100=150" "RF_K4_CL8=1 RF_HYB_R100=95" "RF_K4_CL8=0" "RF_K4_CL8=1 RF_HYB_R100=130"; do
  env $v timeout 300 python scripts/k4_energy.py --gm 8 --reps 6 2>&1 | grep rand | sed "s/^/$v /"; done
