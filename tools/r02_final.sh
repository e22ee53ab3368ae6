#!/bin/bash
# round-end evidence: full GPU suite, default bench line, every config / precision
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/gpu_tests.log 2>&1
tail -3 gpurun_out/gpu_tests.log
python bench.py > gpurun_out/bench_c3_fp64.json 2> gpurun_out/bench_c3_fp64.err
tail -c 300 gpurun_out/bench_c3_fp64.json
bash tools/bench_all.sh
