ncu --set full --import-source on --clock-control none -k regex:k_pc_tri_reg -c 1 -s 2 -o gpurun_out/tri_reg_k128 python scripts/k5_tri_prof.py 128 > gpurun_out/ncu_tri.log 2>&1
ncu -i gpurun_out/tri_reg_k128.ncu-rep --page source --csv --print-source sass > gpurun_out/tri_src.csv 2>&1
ncu -i gpurun_out/tri_reg_k128.ncu-rep --page details --csv > gpurun_out/tri_details.csv 2>&1
