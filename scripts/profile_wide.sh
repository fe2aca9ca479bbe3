#!/bin/bash
# ncu capture of the wide K1 tile (cluster pairs, N = 384) at the C3 fp32-split shape
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_gemm_av_tc -s 3 -c 1 -o gpurun_out/k1_wide_c3 \
    python scripts/one_gemm.py 65536 128 > gpurun_out/ncu_wide.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_gemm_av_tc --csv \
    --log-file gpurun_out/k1_wide_c3_launches.csv python scripts/one_gemm.py 65536 128 > /dev/null 2>&1
ls -la gpurun_out | tail -5
