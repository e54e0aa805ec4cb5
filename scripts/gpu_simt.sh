# SIMT (K6) rewrite: fp32 / fp64 parity, then configs[1] per-mode timings.
timeout 900 python -m pytest tests -m gpu -q -x -k "fp32 or fp64 or config1 or simt or small or ragged or center or acts" 2>&1 | tail -2
bash scripts/gpu_modes_c1.sh
