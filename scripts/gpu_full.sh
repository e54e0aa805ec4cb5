# Full GPU suite, smoke, default bench line (configs[3] step + TRF + configs[4] Φ), with K5 A/B at configs[4].
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 400 gpurun_out/bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench.json").read().strip().splitlines()[-1])
k = d["kernels"]
print("value", round(d["value"], 1), "ms", round(d["ms_per_step"], 2), "launches", d["gpu_launches"], "clocks", d["clocks"])
print({n: (round(v["avg_ms"], 3), round(v.get("achieved_tflops", 0), 1)) for n, v in k.items()})
print("e2e", round(d["e2e"]["value"], 1), d["e2e"]["ms_per_step"])
print("trf", {a: d["trf"][a] for a in ("ms_per_step", "tflops", "K4_ter_tflops_fp8")})
print("phi4", {a: d["phi_configs4"][a] for a in ("ms_per_step", "K5_ms", "K5_hbm_gbs", "K5_frac_hbm")})
PY
