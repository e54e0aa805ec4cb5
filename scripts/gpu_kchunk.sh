# K-chunked accumulation in TMEM: 3xTF32 parity/mainloop tests, then K4 cost vs chunk size at configs[1] shape.
timeout 900 python -m pytest tests -m gpu -q -x -k "3xtf32 or mainloop or packed or chunk" 2>&1 | tail -2
for kc in 4 0 8; do
  echo -n "RF_KCHUNK=$kc: "
  RF_KCHUNK=$kc timeout 600 python bench.py --config 1 --prec 3xtf32 --no-trf --no-phi4 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print({n:(round(v['avg_ms'],3), round(v.get('achieved_tflops',0),1)) for n,v in k.items() if n[:2] in ('K3','K4','K5')})"
done
