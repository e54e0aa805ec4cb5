for mc in 0 1 0 1; do RF_K4TER_MC=$mc timeout 300 python scripts/trf_bench.py --eps 0.9 2>&1 | grep TRF | sed "s/^/mc=$mc /"; done
RF_K4TER_MC=1 timeout 600 python -m pytest tests/test_gpu_trf.py -q 2>&1 | tail -1
