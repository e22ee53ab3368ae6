#!/bin/bash
# GW (32x512, r > 256) launches of the TIMED configuration's kernel, on the product-compress c3 tree
# scaled to N=2^18 (same d/m/s/budget/r): launch list of one evaluation, then ncu --set full with
# source of the output launch and of the largest downward launch; summaries written on the box.
set -u
mkdir -p gpurun_out /tmp/prof
N=${1:-262144}
python tools/profile_run.py --n $N --tree compress --evals 1 > gpurun_out/gw_r02_run.log 2>&1
[ -f gpurun_out/gw_r02_launches.csv ] || timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k "regex:grouped_gemm_f64" --csv --log-file gpurun_out/gw_r02_launches.csv \
    python tools/profile_run.py --n $N --tree compress --evals 1 > /dev/null 2>&1
echo "launch list rc=$?"
# the GW launches of one evaluation: output = the last one; downward leaf level = the one before it
# grouped-GEMM launches of one evaluation: upward levels depth..1, downward 1..depth, output; the
# last two are the leaf-level downward (S2S + S2N) and the output (L2L + leaf S2N) GW launches
NG=$(grep -c "grouped_gemm_f64" gpurun_out/gw_r02_launches.csv)
NG=$((NG / 4))
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:grouped_gemm_f64" \
    --launch-skip $((NG-2)) --launch-count 2 \
    -o /tmp/prof/gw python tools/profile_run.py --n $N --tree compress --evals 1 > gpurun_out/gw_r02_ncu.log 2>&1
echo "full capture rc=$?"
ncu -i /tmp/prof/gw.ncu-rep --page raw --csv --metrics gpu__time_duration.sum > /tmp/prof/ids.csv 2>&1
NL=$(grep -c "grouped_gemm" /tmp/prof/ids.csv)
echo "gw launches: $NL"
for k in $((NL-1)) $((NL-2)); do
  ncu -i /tmp/prof/gw.ncu-rep --launch-skip $k --launch-count 1 --page source --csv --print-source sass > /tmp/prof/src_$k.csv 2>&1
  python tools/ncu_source_top.py /tmp/prof/src_$k.csv 50 > gpurun_out/gw_r02_src_$k.txt 2>&1
  ncu -i /tmp/prof/gw.ncu-rep --launch-skip $k --launch-count 1 --page details --csv > gpurun_out/gw_r02_details_$k.csv 2>&1
  ncu -i /tmp/prof/gw.ncu-rep --launch-skip $k --launch-count 1 --page raw --csv > gpurun_out/gw_r02_raw_$k.csv 2>&1
done
cp /tmp/prof/gw.ncu-rep gpurun_out/gw_r02.ncu-rep 2>/dev/null
ls -la gpurun_out/gw_r02.ncu-rep
echo done
