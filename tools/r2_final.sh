# (bounds-checked build rebuilt first: FLMISR_LIB=build_variants/lib_bounds.so FLMISR_DEFS=-DFLMISR_BOUNDS python -m paper_2108_04315_b200.build)
# round-2 final evidence on one GPU: full GPU suite, bounds-checked streaming suites (incl. det mode),
# bench lines of every config, smoke, C3 launch list and one ncu --set full capture of the loop kernel
set -u
python -m pytest tests -m gpu -q > gpurun_out/final_gpu_tests.log 2>&1; echo "exit=$?" >> gpurun_out/final_gpu_tests.log
FLMISR_LIB=$PWD/build_variants/lib_bounds.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_pc.py tests/test_gpu_bands.py tests/test_gpu_pipeline.py tests/test_gpu_fullsize.py tests/test_gpu_det.py tests/test_gpu_threads.py -m gpu -q > gpurun_out/final_bounds_tests.log 2>&1; echo "exit=$?" >> gpurun_out/final_bounds_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "exit=$?" >> gpurun_out/final_smoke.log
python bench.py > gpurun_out/final_bench_C3.log 2>&1
python bench.py --config C2 --no-cpu-baseline > gpurun_out/final_bench_C2.log 2>&1
python bench.py --config C4 --no-cpu-baseline > gpurun_out/final_bench_C4.log 2>&1
python bench.py --config C6 --no-cpu-baseline --steps 20 > gpurun_out/final_bench_C6.log 2>&1
python bench.py --config G3 --no-cpu-baseline --steps 20 > gpurun_out/final_bench_G3.log 2>&1
python bench.py --mode stream --steps 40 > gpurun_out/final_bench_C5.log 2>&1
python bench.py --mode stream --u16 --steps 40 > gpurun_out/final_bench_C5u16.log 2>&1
python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/final_bench_ref.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches_C3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/final_ncu_launch_C3.log 2>&1
ncu --set full --clock-control none -k regex:k_scg_loop -c 1 --csv --page raw python tools/profile_step.py --config C3 --reps 1 > gpurun_out/final_ncu_full_C3.csv 2> gpurun_out/final_ncu_full_C3.err
