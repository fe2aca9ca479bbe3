#!/bin/bash
# Profiles committed under profiles/ (run on the GPU box from the repo root):
#  * launch list of the bench command (per-kernel durations, cold-cache, serialised)
#  * ncu --set full of the top kernels at C2 shape (and the fp64 Hessenberg at C3 shape)
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 800 --csv \
    --log-file gpurun_out/launches_c2_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gemm_av_tc -s 2 -c 1 -o gpurun_out/k1_c2 python scripts/one_gemm.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_ozk_gemm -c 1 -o gpurun_out/ozk_gemm_c2 python scripts/one_resid.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gram_partial -s 2 -c 1 -o gpurun_out/gram_c2 python scripts/one_gram.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_hessenberg -s 1 -c 1 -o gpurun_out/hess_c2 python scripts/micro_hess.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pc_tri_reg -s 2 -c 1 -o gpurun_out/pc_tri_k64 python scripts/pc_phases.py 64 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pc_eigvec -s 2 -c 1 -o gpurun_out/pc_eigvec_k64 python scripts/pc_phases.py 64 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pc_chol -s 2 -c 1 -o gpurun_out/pc_chol_k64 python scripts/pc_phases.py 64 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_resid_est -c 1 -o gpurun_out/resid_est_c2 python bench.py --config c2 --steps 2 --warmup 1 --no-cpu > /dev/null 2>&1
ls -la gpurun_out
