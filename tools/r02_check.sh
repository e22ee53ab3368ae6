#!/bin/bash
# Round-2 state check: GPU suite + default bench line (product-compress c3 tree) + reference arm.
set -u
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/r02_box.txt 2>&1; nproc >> gpurun_out/r02_box.txt; free -g >> gpurun_out/r02_box.txt
timeout 1500 python -m pytest tests -m gpu -q -x --durations=25 > gpurun_out/r02_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/r02_gpu_tests.log
timeout 1200 python bench.py > gpurun_out/r02_bench_c3.json 2> gpurun_out/r02_bench_c3.err; echo "bench rc=$?"; tail -1 gpurun_out/r02_bench_c3.json | cut -c1-400; tail -5 gpurun_out/r02_bench_c3.err
