#!/bin/bash
# End-of-round measurement (outputs in gpurun_out/, copied into profiles/ by hand): the GPU test
# suite, every config's bench line, the default bench line, the reference arm, the launch list
# of the default bench command, and the §8(f) benches (skeletonisation, ANN).
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/final_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/final_gpu_tests.log
bash tools/bench_all.sh
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -1 gpurun_out/bench_c3.json | cut -c1-200
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -1 gpurun_out/bench_ref.json | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_launches.log 2>&1; echo "launch list rc=$?"
timeout 600 python tools/bench_skel.py > gpurun_out/skel_bench.json 2>&1; tail -1 gpurun_out/skel_bench.json | cut -c1-200
timeout 600 python tools/bench_ann.py > gpurun_out/ann_bench.json 2>&1; tail -1 gpurun_out/ann_bench.json | cut -c1-200
