#!/bin/bash
# PDL change: parity subset, c1/c2 latency with and without PDL, default bench line.
mkdir -p gpurun_out
python -m pytest tests/test_parity_gpu.py tests/test_golden.py tests/test_boundary_gpu.py tests/test_parity_configs_gpu.py -q -x > gpurun_out/pdl_tests.log 2>&1
tail -3 gpurun_out/pdl_tests.log
for c in c1 c2; do
  python tools/latency_probe.py $c --reps 100 > gpurun_out/lat_${c}_pdl.json 2> gpurun_out/lat_${c}_pdl.err
  GOFMM_NO_PDL=1 python tools/latency_probe.py $c --reps 100 > gpurun_out/lat_${c}_nopdl.json 2> gpurun_out/lat_${c}_nopdl.err
done
python - <<'PY'
import json
for c in ("c1", "c2"):
    for v in ("pdl", "nopdl"):
        try:
            d = json.load(open(f"gpurun_out/lat_{c}_{v}.json"))
            print(c, v, d["graph_ms_median"], d["tflops"], d["timed_phase_ms"])
        except Exception as e:
            print(c, v, "failed", e)
PY
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
tail -c 600 gpurun_out/bench_c3.json
