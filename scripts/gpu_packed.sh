# RF_OUT_PACKED_TRI parity, the full GPU suite, and the pipelined e2e bench line.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-phi4 --no-trf > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err
tail -c 800 gpurun_out/bench_e2e.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_e2e.json").read().strip().splitlines()[-1])
print("value", d["value"], "ms", d["ms_per_step"], "launches", d["gpu_launches"], "e2e", json.dumps(d["e2e"]))
PY
