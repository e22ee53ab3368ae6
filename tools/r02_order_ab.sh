#!/bin/bash
# A/B of the tile order of many-wave launches on the FULL c3 product-compress tree: per-launch device
# times (CUDA events) and ncu DRAM bytes of the leaf-level downward and output launches.
mkdir -p gpurun_out
for W in 4 1000000; do
  GOFMM_TREE_ORDER_WAVES=$W python tools/profile_run.py --n 1048576 --tree compress --evals 2 2>&1 \
      | grep -E "^1 |level  1[01]|output" | cut -c1-220 | sed "s/^/[waves=$W] /"
  GOFMM_TREE_ORDER_WAVES=$W timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
      --clock-control none -k "regex:grouped_gemm_f64" --launch-skip 20 --launch-count 3 --csv \
      --log-file gpurun_out/order_ab_$W.csv python tools/profile_run.py --n 1048576 --tree compress --evals 1 > /dev/null 2>&1
  python - $W <<'PY'
import csv, sys
w = sys.argv[1]
rows = [r for r in csv.reader(open(f"gpurun_out/order_ab_{w}.csv")) if len(r) > 10 and r[0].isdigit()]
for r in rows:
    print(f"[waves={w}] launch {r[0]} {r[4][:45]} {r[12]} = {r[14]} {r[13]}")
PY
done
