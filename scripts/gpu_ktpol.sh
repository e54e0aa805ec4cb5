# K̃ operand-load L2 policy (RF_KT_LOADPOL), interleaved; then the GPU suite.
for i in 1 2 3; do for v in 0 1; do echo -n "kt_pol=$v "; RF_KT_LOADPOL=$v timeout 300 python scripts/center_bench.py 2>&1 | grep "K̃" | cut -c1-70 | tr '\n' ' '; echo; done; done
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
