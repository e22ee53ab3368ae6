#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_golden.py tests/test_parity_gpu.py tests/test_boundary_gpu.py tests/test_parity_configs_gpu.py tests/test_adapter_gpu.py -q -x 2>&1 | tail -4
python tools/profile_run.py --n 262144 --tree compress --evals 2 2>&1 | grep -E "^1 |level   [89]|output" | cut -c1-200
python tools/latency_probe.py c1 --reps 100 > gpurun_out/lat_c1.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/lat_c1.json'));print('c1', d['graph_ms_median'], d['tflops'], d['timed_phase_ms'])"
