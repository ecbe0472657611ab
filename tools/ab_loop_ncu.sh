# loop-kernel A/B under ncu (one launch holds all phases, so cross-phase L2 reuse is measured)
for L in paper_2108_04315_b200/libflmisr.so build_variants/lib_up.so; do
FLMISR_LIB=$PWD/$L ncu --clock-control none -k regex:k_scg_loop -s 3 -c 1 \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_lookup_hit.sum,lts__t_sectors_lookup_miss.sum \
  --csv python tools/tune.py --reps 1 > gpurun_out/abl_$(basename $L .so).csv 2>&1
done
LIBS="paper_2108_04315_b200/libflmisr.so build_variants/lib_up.so" bash tools/ab.sh > gpurun_out/ab.log 2>&1
