# K4^ter (fp8) hybrid with 4-CTA vs 8-CTA multicast clusters (RF_K4_CL8), interleaved; bit-exactness of G^ter.
for v in 0 1 0 1; do echo -n "RF_K4_CL8=$v: "; RF_K4_CL8=$v timeout 300 python scripts/trf_bench.py --eps 0.9 --reps 6 2>&1 | grep TRF | cut -c60-200; done
RF_K4_CL8=1 timeout 300 python -m pytest tests/test_gpu_trf.py -m gpu -q -x 2>&1 | tail -1
