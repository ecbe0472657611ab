set -x
ncu --set full --import-source on --clock-control none -k regex:k_scg_loop4 -c 1 -o gpurun_out/r2_g3_loop -f python tools/profile_step.py --config G3 --reps 1 > gpurun_out/r2_ncu_g3_loop.log 2>&1
M=gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active
FLMISR_NO_PERSIST=1 ncu --clock-control none -k regex:"k_vg4|k_uc4" -s 2 -c 4 --metrics $M --csv python tools/profile_step.py --config G3 --reps 1 > gpurun_out/r2_ncu_g3_phases.csv 2>&1
FLMISR_NO_PERSIST=1 ncu --clock-control none -k regex:"k_vg_stream|k_uc_stream" -s 2 -c 4 --metrics $M --csv python tools/profile_step.py --config C3 --reps 1 > gpurun_out/r2_ncu_c3_phases.csv 2>&1
