# A/B: committed build (librf_b200_old.so, experiments only) vs the working tree: K5 at configs[4] / configs[3]
# shapes and the K3+K4 loop, interleaved; then the GPU parity suite of the working tree.
L=$PWD/paper_2110_01899_b200
for i in 1 2; do
  for v in old new; do
    f=$L/librf_b200.so; [ $v = old ] && f=$L/librf_b200_old.so
    echo -n "$v c4: "; RF_B200_LIB=$f timeout 300 python scripts/k5_bench.py --reps 5 2>&1 | tail -1 | cut -c1-90
    echo -n "$v c3: "; RF_B200_LIB=$f timeout 300 python scripts/k5_bench.py --n 65536 --p 1024 --reps 5 2>&1 | tail -1 | cut -c1-90
    echo -n "$v k34: "; RF_B200_LIB=$f timeout 300 python scripts/k4_energy.py --gm 8 --reps 6 2>&1 | grep rand | cut -c1-110
  done
done
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
