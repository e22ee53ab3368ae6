#!/bin/bash
# full GPU suite + default bench line + FP32 bench line
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/gpu_tests.log 2>&1
tail -14 gpurun_out/gpu_tests.log
python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
tail -c 400 gpurun_out/bench_c3.json
python bench.py --precision fp32 --no-cpu > gpurun_out/bench_c3_fp32.json 2> gpurun_out/bench_c3_fp32.err
tail -c 400 gpurun_out/bench_c3_fp32.json
