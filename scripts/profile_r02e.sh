#!/bin/bash
# Late round-2 refresh (default bench config c3-ladder3l): the per-kernel launch list with DRAM
# bytes, and an ncu capture of the K7z row-scale prepare at 128 threads per row.
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu --no-table"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c3_bench.csv $B > gpurun_out/ncu_launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_oz_rowscale -s 1 -c 1 \
    -o gpurun_out/oz_rowscale_c3 $B > gpurun_out/ncu_oz_rowscale_c3.log 2>&1
ls -la gpurun_out | tail -5
