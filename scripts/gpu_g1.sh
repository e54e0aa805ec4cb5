# G1 (rf_round_bf16): its GPU parity tests, smoke, and the default bench line with G1 inside the step.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_round.py -q > gpurun_out/g1_tests.log 2>&1; tail -3 gpurun_out/g1_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1_smoke.log 2>&1; tail -3 gpurun_out/g1_smoke.log
timeout 900 python bench.py > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err; tail -3 gpurun_out/g1_bench.err
python - <<'P'
import json
d = json.loads(open("gpurun_out/g1_bench.json").read().strip().splitlines()[-1])
print("value", d["value"], "e2e", d["e2e"]["value"], "h2d", d["e2e"]["h2d_bytes_per_step"], "launches", d["gpu_launches"],
      d["e2e"]["gpu_launches"], "ms", d["ms_per_step"], {k: v["avg_ms"] for k, v in d["kernels"].items() if "G1" in k or "K1" in k})
P
