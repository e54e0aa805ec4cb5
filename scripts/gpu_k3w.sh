# K3 with 8 vs 12 epilogue warps at configs[3] (bench step without extras), interleaved.
for v in 0 1 0 1; do
  echo -n "RF_K3_WIDE=$v: "
  RF_K3_WIDE=$v timeout 600 python bench.py --steps 3 --no-trf --no-phi4 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print(round(d['value'],1), {n:(round(v['avg_ms'],3), round(v.get('achieved_tflops',0),1)) for n,v in k.items() if n[:2] in ('K3','K5') or n=='K4_syrk'})"
done
timeout 600 python -m pytest tests -m gpu -q -x -k "ktilde or center" 2>&1 | tail -1
RF_K3_WIDE=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_acts.py -m gpu -q -x 2>&1 | tail -1
