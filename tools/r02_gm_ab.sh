#!/bin/bash
for e in 0.74 0.72; do
  GOFMM_GM_EFF=$e python tools/latency_probe.py c2 --reps 20 > gpurun_out/l2_$e.json 2> gpurun_out/l2_$e.err
  tail -2 gpurun_out/l2_$e.err
  python - $e <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/l2_{sys.argv[1]}.json"))
print("c2 gm_eff", sys.argv[1], d["graph_ms_median"], d["timed_phase_ms"]["ms_output"], d["timed_phase_ms"]["ms_downward"])
PY
done
