#!/bin/bash
# ncu captures of the K7z tiers added late in round 2 (default bench config): the 3-level entry
# pass (k_ozk_ts<.,128,3>) and the 5-level lead pass (k_ozk_ts<.,64,5>), plus the 1-slice K1 start pass.
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu --no-table"
# launch order per solve: k_ozk_ts<.,128,3> x2 (entry pass, entry projection), <.,64,5> x2 (lead),
# <.,64,6> x2; k_gemm_av_tc: the 1-slice start pass first
for spec in "k_ozk_ts:0:ozk_ts3_c3" "k_ozk_ts:2:ozk_ts5_c3" "k_gemm_av_tc:0:k1_start_c3"; do
  IFS=: read -r kern skip name <<< "$spec"
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$kern" -s $skip -c 1 \
      -o gpurun_out/$name $B > gpurun_out/ncu_$name.log 2>&1
done
ls -la gpurun_out/*.ncu-rep | tail -3
