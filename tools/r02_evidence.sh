#!/bin/bash
# round-end evidence on the final code: GPU suite, default bench line, every config / precision,
# the ncu launch list of the default bench command (shares of the step per kernel)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/box.txt
python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/gpu_tests.log 2>&1
tail -1 gpurun_out/gpu_tests.log
python bench.py > gpurun_out/bench_c3_fp64.json 2> gpurun_out/bench_c3_fp64.err
tail -c 300 gpurun_out/bench_c3_fp64.json
bash tools/bench_all.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_c3.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_bench.log 2>&1
echo "ncu rc=$?"
python tools/launch_shares.py gpurun_out/launches_c3.csv > gpurun_out/launch_shares_c3.txt 2>&1
head -12 gpurun_out/launch_shares_c3.txt
