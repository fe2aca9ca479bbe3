#!/bin/bash
# Round-2 profiles of the default bench config (C3 headline, c3-ladder3l), run on the GPU box
# from the repo root; summaries -> profiles/ via scripts/summarize_profiles.py r02b.
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu --no-table"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c3_bench.csv $B > gpurun_out/ncu_launches.log 2>&1
for spec in "k_gemm_av_tc:6:k1_c3" "k_ozk_ts:2:ozk_ts_c3" "k_ozk_gemm:1:ozk_lite_c3" "k_restart_dmma:2:restart_c3" \
            "k_pc_chol_blk:2:chol_blk_k128" "k_pc_tri_reg:2:pc_tri_k128" "k_gram_partial:2:gram_c3"; do
  IFS=: read -r kern skip name <<< "$spec"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$kern -s $skip -c 1 \
      -o gpurun_out/$name $B > gpurun_out/ncu_$name.log 2>&1
done
ls -la gpurun_out | tail -12
