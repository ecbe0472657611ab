# per-phase VG/UC kernels of two builds under ncu (cold L2 per kernel): intrinsic cost of the code
for L in paper_2108_04315_b200/libflmisr.so build_variants/lib_up.so; do
FLMISR_LIB=$PWD/$L FLMISR_NO_PERSIST=1 ncu --clock-control none -k regex:"k_vg_stream|k_uc_stream" -s 20 -c 4 \
  --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio \
  --csv python tools/tune.py --reps 1 > gpurun_out/abv_$(basename $L .so).csv 2>&1
done
