# Default bench (with the configs[4] bf16/tf32/3xtf32 Φ object) and a 3xtf32 configs[1] line (fp32-accurate mode).
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 300 gpurun_out/bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench.json").read().strip().splitlines()[-1])
print("value", round(d["value"], 1), "e2e", round(d["e2e"]["value"], 1))
p4 = d["phi_configs4"]
for k in ("ms_per_step", "K5_ms", "K5_hbm_gbs"):
    print(k, p4[k], p4["tf32"][k], p4["3xtf32"][k])
PY
timeout 600 python bench.py --config 1 --prec 3xtf32 --no-trf --no-phi4 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; tail -c 300 gpurun_out/bench_c1.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_c1.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline'], d['peaks'])"
