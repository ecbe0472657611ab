# A/B of tuning builds: per-reconstruction loop-kernel time (and per-phase kernels) on C3-sized random stacks
LIBS=${LIBS:-"paper_2108_04315_b200/libflmisr.so build_variants/lib_down.so build_variants/lib_orig.so"}
for i in 1 2; do
for L in $LIBS; do
FLMISR_LIB=$PWD/$L python tools/tune.py --reps 20
[ -n "$PERPHASE" ] && FLMISR_LIB=$PWD/$L FLMISR_NO_PERSIST=1 python tools/tune.py --reps 20
done; done
