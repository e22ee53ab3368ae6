#!/bin/bash
# final code: full GPU suite, smoke, the FP32 c1 / c2 bench lines (after the FP32 pre-wait change)
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/gpu_tests.log 2>&1
tail -1 gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --config c1 --precision fp32 --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_c1_fp32.json 2> gpurun_out/bench_c1_fp32.err
timeout 900 python bench.py --config c2 --precision fp32 --steps 10 --warmup 3 > gpurun_out/bench_c2_fp32.json 2> gpurun_out/bench_c2_fp32.err
tail -c 200 gpurun_out/bench_c2_fp32.json
