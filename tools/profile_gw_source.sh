#!/bin/bash
# Source-level stall attribution of the GW output launch (c3-shaped, N=2^18): ncu --set full with
# source import of every GW launch of one evaluation; the last one (the output launch) is
# summarised on the box.
set -u
mkdir -p gpurun_out /tmp/prof
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:grouped_gemm_f64<\(int\)32" --launch-count 20 \
    -o /tmp/prof/gw_all python tools/profile_run.py --n 262144 --evals 1 > gpurun_out/ncu_gw_src.log 2>&1
echo "capture rc=$?"
ncu -i /tmp/prof/gw_all.ncu-rep --page raw --csv --metrics gpu__time_duration.sum > /tmp/prof/ids.csv 2>&1
NL=$(grep -c "grouped_gemm" /tmp/prof/ids.csv)
echo "gw launches: $NL"
ncu -i /tmp/prof/gw_all.ncu-rep --launch-skip $((NL-1)) --launch-count 1 --page source --csv --print-source sass \
    > /tmp/prof/gw_src.csv 2>&1
python tools/ncu_source_top.py /tmp/prof/gw_src.csv 60 > gpurun_out/ncu_gw_out_source_top.txt 2>&1
ncu -i /tmp/prof/gw_all.ncu-rep --launch-skip $((NL-1)) --launch-count 1 --page details --csv \
    > gpurun_out/ncu_gw_out_details.csv 2>&1
head -c 3000 /tmp/prof/gw_src.csv > gpurun_out/gw_src_head.csv
echo done
