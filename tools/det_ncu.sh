for T in 6; do
  DET_ROWS=$T ncu --set full --import-source on --clock-control none -k regex:k_scg_loop -c 1 -f -o gpurun_out/det_T$T python tools/det_profile.py > gpurun_out/det_ncu_T$T.log 2>&1
  ncu -i gpurun_out/det_T$T.ncu-rep --page source --csv --print-source sass > gpurun_out/det_src_T$T.csv 2>&1
  ncu -i gpurun_out/det_T$T.ncu-rep --page source --csv --print-source cuda > gpurun_out/det_srccu_T$T.csv 2>&1
  rm -f gpurun_out/det_T$T.ncu-rep
done
DET_ROWS=0 ncu --set full --import-source on --clock-control none -k regex:k_scg_loop -c 1 -f -o gpurun_out/det_T0 python tools/det_profile.py > gpurun_out/det_ncu_T0.log 2>&1
ncu -i gpurun_out/det_T0.ncu-rep --page source --csv --print-source sass > gpurun_out/det_src_T0.csv 2>&1
ncu -i gpurun_out/det_T0.ncu-rep --page source --csv --print-source cuda > gpurun_out/det_srccu_T0.csv 2>&1
rm -f gpurun_out/det_T0.ncu-rep
