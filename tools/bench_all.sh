#!/bin/bash
# Every BASELINE.json config through bench.py (fp64; fp32 where BASELINE names it), one JSON
# line each under gpurun_out/bench_<config>_<precision>.json. Run on the GPU box via gpurun.
set -u
mkdir -p gpurun_out
run() {  # config precision steps extra...
  local c=$1 p=$2 k=$3; shift 3
  timeout 1200 python bench.py --config "$c" --precision "$p" --steps "$k" --warmup 3 "$@" \
    > "gpurun_out/bench_${c}_${p}.json" 2> "gpurun_out/bench_${c}_${p}.err"
  echo "$c $p rc=$?"; tail -1 "gpurun_out/bench_${c}_${p}.json" | cut -c1-160
}
run c1 fp64 20
run c1 fp32 20 --no-cpu
run c2 fp64 10
run c2 fp32 10
run c4 fp64 5
run c4 fp32 5 --no-cpu
run c3 fp32 5
run c5 fp64 3 --no-cpu --e2e-steps 1
run c5 fp32 3 --no-cpu --e2e-steps 1
