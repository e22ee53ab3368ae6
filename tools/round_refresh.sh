#!/bin/bash
# Refresh every measured artefact of the round (outputs in gpurun_out/; copied to profiles/ by hand):
# ncu --set full summary of the GW launches at N=2^18, every config's bench line, the default
# bench line and the reference arm.
set -u
mkdir -p gpurun_out /tmp/prof
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:grouped_gemm_f64<\(int\)32" --launch-count 10 \
    -o /tmp/prof/c3n18_wide python tools/profile_run.py --n 262144 --evals 1 > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
python tools/ncu_summary.py /tmp/prof/c3n18_wide.ncu-rep > gpurun_out/ncu_c3n18_wide_summary.txt 2>&1
ncu -i /tmp/prof/c3n18_wide.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active > gpurun_out/ncu_c3n18_wide_raw.csv 2>&1
bash tools/bench_all.sh
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -1 gpurun_out/bench_c3.json | cut -c1-200
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -1 gpurun_out/bench_ref.json | cut -c1-200
