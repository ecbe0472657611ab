# per-phase path: parity + phase metrics + G3 bench (one GPU)
python -m pytest tests/test_gpu_pc.py -q -x > gpurun_out/pc_tests.log 2>&1; echo "exit=$?" >> gpurun_out/pc_tests.log
M=gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread
FLMISR_NO_PERSIST=1 ncu --clock-control none -k regex:"k_vg4|k_uc4" -s 2 -c 2 --metrics $M --csv python tools/profile_step.py --config G3 --reps 1 > gpurun_out/pc_phases.csv 2>&1
python bench.py --config G3 --no-cpu-baseline --steps 10 > gpurun_out/pc_g3.log 2>&1
