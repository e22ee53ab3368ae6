#!/bin/bash
# quick A/B of a kernel change: parity subset, GW launch rates on the N=2^18 product-compress c3
# tree, c1 latency
mkdir -p gpurun_out
python -m pytest tests/test_golden.py tests/test_parity_gpu.py -q -x 2>&1 | tail -2
python tools/profile_run.py --n 262144 --tree compress --evals 2 2>&1 | grep -E "^1 |level   [89]|output" | cut -c1-200
python tools/latency_probe.py c1 --reps 100 > gpurun_out/lat_c1.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/lat_c1.json'));print('c1', d['graph_ms_median'], d['tflops'])"
