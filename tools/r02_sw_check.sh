#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_golden.py tests/test_parity_gpu.py tests/test_parity_configs_gpu.py -q -x 2>&1 | tail -2
for c in c5 c2 c1; do
  python tools/latency_probe.py $c --reps 10 > gpurun_out/lat_${c}_sw.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/lat_${c}_sw.json'));print('$c', d['graph_ms_median'], d['tflops'], d['timed_phase_ms'])"
done
python tools/profile_run.py --n 262144 --tree compress --evals 2 2>&1 | grep -E "^1 " | cut -c1-200
