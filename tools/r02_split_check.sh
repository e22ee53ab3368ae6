#!/bin/bash
# A/B of a latency-path change: parity subset (FP64 + FP32), c1 / c2 graph latency per launch
mkdir -p gpurun_out
python -m pytest tests/test_golden.py tests/test_parity_gpu.py tests/test_parity_gpu_f32.py -q -x 2>&1 | tail -2
for c in c1 c2; do
  for p in fp64 fp32; do
    python tools/latency_probe.py $c --reps 100 --precision $p > gpurun_out/lat3_${c}_$p.json 2>/dev/null
    python - "$c" "$p" <<'PY'
import json, sys
c, p = sys.argv[1], sys.argv[2]
d = json.load(open(f"gpurun_out/lat3_{c}_{p}.json"))
print(c, p, d["graph_ms_median"], d["tflops"], " ".join(f"{L['phase'][0]}{L['level']}:{L['ctas']}/{L['ms']}" for L in d["launches"]))
PY
  done
done
