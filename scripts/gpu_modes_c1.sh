# configs[1] (p = 784, n = 4096, m = 8192) in each precision mode: per-kernel times and rates.
for prec in fp32 3xtf32 tf32 bf16; do
  echo -n "$prec: "
  timeout 600 python bench.py --config 1 --prec $prec --no-trf --no-phi4 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print(round(d['value'],1), round(d['ms_per_step'],3), {n:(round(v['avg_ms'],3), round(v.get('achieved_tflops',0),1)) for n,v in k.items() if v['avg_ms']>0.02})"
done
