# K̃ epilogue-warp variants (env switches), interleaved, + parity of the K5 16-warp default.
for v in "RF_KT_W16=0" "RF_KT_W16=1" "RF_KT_S1=1" "RF_KT_W16=0" "RF_KT_W16=1" "RF_KT_S1=1"; do echo "$v"; env $v timeout 600 python scripts/center_bench.py 2>&1 | grep "K̃"; done
RF_KT_W16=1 timeout 600 python -m pytest tests -m gpu -q -x -k "ktilde or center or phi or Phi or eq1 or packed_tri" 2>&1 | tail -1
