#!/bin/bash
# Round-2 (late) ncu captures of the kernels changed after profiles/r02b_*, default bench config.
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu --no-table"
for spec in "k_restart_dmma:2:restart_c3" "k_oz_resid:4:oz_resid_c3" "k_gram_partial:6:gram_f64_c3" \
            "k_hessenberg:6:hess_f64_c3" "k_oz_slices_vs:2:oz_slices_c3"; do
  IFS=: read -r kern skip name <<< "$spec"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$kern -s $skip -c 1 \
      -o gpurun_out/$name $B > gpurun_out/ncu_$name.log 2>&1
done
ls -la gpurun_out/*.ncu-rep | tail -6
