#!/bin/bash
# Round-1 re-measurement after the wide generated-operand config (outputs in gpurun_out/):
#   1. ncu launch list of the bench command (cold-cache, serialised: compare shares)
#   2. ncu --set full of the wide generated-operand launches of one c3-shaped evaluation at
#      N=2^18, summarised on the box (tools/ncu_summary.py; the report itself stays there)
#   3. DRAM bytes of every grouped GEMM launch at full c3 size
set -u
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"
mkdir -p /tmp/prof
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:grouped_gemm_f64<\(int\)32" --launch-count 10 \
    -o /tmp/prof/c3n18_wide python tools/profile_run.py --n 262144 --evals 1 > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"; tail -2 gpurun_out/ncu_full.log
python tools/ncu_summary.py /tmp/prof/c3n18_wide.ncu-rep > gpurun_out/ncu_c3n18_wide_summary.txt 2>&1
echo "summary rc=$?"
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum \
    --clock-control none -k regex:grouped_gemm_f64 --csv --log-file gpurun_out/dram_c3.csv \
    python tools/profile_run.py --n 1048576 --evals 1 > gpurun_out/ncu_dram.log 2>&1
echo "dram rc=$?"
