# The full bench line (TRF included) in every precision mode on the small configs, one line each.
for a in "--config 0 --prec fp64" "--config 1 --prec fp32" "--config 1 --prec 3xtf32" "--config 1 --prec tf32" "--config 2"; do
  echo -n "$a: "; timeout 600 python bench.py $a --steps 3 --no-cpu-baseline 2>/tmp/err.log | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],2), d['unit'], 'e2e', round(d['e2e']['value'],2), d['e2e']['d2h_bytes_per_step'], d['dtype'], 'trf', d['trf'] and round(d['trf']['tflops'],1))" || tail -3 /tmp/err.log
done
