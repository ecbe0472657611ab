# A/B of per-phase kernel builds: phase metrics and G3 bench per library
M=gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread
for L in paper_2108_04315_b200/libflmisr.so build_variants/lib_wpb16.so; do
  n=$(basename $L .so)
  FLMISR_LIB=$PWD/$L FLMISR_NO_PERSIST=1 ncu --clock-control none -k regex:"k_vg4|k_uc4" -s 2 -c 2 --metrics $M --csv python tools/profile_step.py --config G3 --reps 1 > gpurun_out/ab_$n.csv 2>&1
  FLMISR_LIB=$PWD/$L python bench.py --config G3 --no-cpu-baseline --steps 10 > gpurun_out/ab_$n.log 2>&1
done
python -m pytest tests/test_gpu_pc.py -q -x > gpurun_out/pc_tests.log 2>&1; echo "exit=$?" >> gpurun_out/pc_tests.log
