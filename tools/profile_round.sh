#!/bin/bash
# Round measurement recipe (run on the GPU box through gpurun; outputs land in gpurun_out/).
#   1. bench.py default line (c3) and the reference arm
#   2. ncu launch list of the bench command (cold-cache, serialised: compare shares)
#   3. ncu --set full of the dominant launches at full c3 size (traffic, pipes, stalls)
set -u
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -1 gpurun_out/bench_c3.json
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -1 gpurun_out/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_launches.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:grouped_gemm --launch-skip 21 --launch-count 2 \
    -o gpurun_out/prof_c3_full python tools/profile_run.py --n 1048576 --evals 1 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
