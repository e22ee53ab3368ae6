#!/bin/bash
# FP32 (3xTF32 tcgen05) measurement recipe, run on the GPU box through gpurun; outputs land in
# gpurun_out/. c3 has 23 grouped-GEMM launches per evaluation (11 N2S, 11 downward, 1 output);
# profile_run.py evaluates twice, so launch 23+21 = 44 is the second evaluation's leaf-level
# downward launch and 45 its output launch.
set -u
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3_f32.csv \
    python bench.py --precision fp32 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_launches_f32.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:tf32x3 --launch-skip 44 --launch-count 2 --csv --log-file gpurun_out/ncu_c3_f32_dram.csv \
    python tools/profile_run.py --n 1048576 --precision fp32 --evals 2 > gpurun_out/ncu_dram_f32.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tf32x3 --launch-skip 37 --launch-count 1 \
    -o gpurun_out/prof_f32_n18 python tools/profile_run.py --n 262144 --precision fp32 --evals 2 > gpurun_out/ncu_full_f32.log 2>&1
tail -2 gpurun_out/ncu_full_f32.log
