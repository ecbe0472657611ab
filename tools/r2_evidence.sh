# round-2 evidence (one GPU): band-size scaling inputs for C3/C4/C6, peer emulation, launch lists, ncu of the G3 loop
python tools/band_size.py --config C3 --reps 10 > gpurun_out/band_C3.json 2>&1
python tools/band_size.py --config C4 --reps 5 > gpurun_out/band_C4.json 2>&1
python tools/band_size.py --config C6 --reps 5 > gpurun_out/band_C6.json 2>&1
python tools/peer_emulation.py > gpurun_out/peer_emu.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_C3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_C3.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_G3.csv python bench.py --config G3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_G3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_scg_loop4 -c 1 -o gpurun_out/r2_g3_loop_final -f python tools/profile_step.py --config G3 --reps 1 > gpurun_out/r2_ncu_g3_loop2.log 2>&1
