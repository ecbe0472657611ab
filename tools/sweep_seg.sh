for lib in paper_2108_04315_b200/libflmisr.so build_variants/lib_w1_m16.so build_variants/lib_w2_m8.so build_variants/lib_w4_m4.so; do
  for S in auto 46 31 19 13; do
    if [ $S = auto ]; then FLMISR_LIB=$lib timeout 120 python tools/tune.py; else FLMISR_LIB=$lib FLMISR_SEG_ROWS=$S timeout 120 python tools/tune.py; fi
  done
done
