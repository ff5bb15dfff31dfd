ncu --set full --clock-control none -k regex:nb_residual_kernel -s 3 -c 1 -o gpurun_out/res_c3 python scripts/resid_variants.py c3 > gpurun_out/ncu_res.log 2>&1
ncu -i gpurun_out/res_c3.ncu-rep --page raw --csv > gpurun_out/res_c3_raw.csv 2>&1
ncu -i gpurun_out/res_c3.ncu-rep --page details --csv > gpurun_out/res_c3_details.csv 2>&1
rm -f gpurun_out/res_c3.ncu-rep
