# round-2 bench lines (one GPU) and the bounds-checked test run
export FLMISR_BOUNDS_LIB=$PWD/build_variants/lib_bounds.so
FLMISR_LIB=$FLMISR_BOUNDS_LIB python -m pytest tests/test_gpu_parity.py tests/test_gpu_pc.py tests/test_gpu_bands.py tests/test_gpu_pipeline.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/bounds_tests.log 2>&1; echo "exit=$?" >> gpurun_out/bounds_tests.log
python bench.py > gpurun_out/bench_C3.log 2>&1
python bench.py --config C2 --no-cpu-baseline > gpurun_out/bench_C2.log 2>&1
python bench.py --config C4 --no-cpu-baseline > gpurun_out/bench_C4.log 2>&1
python bench.py --config C6 --no-cpu-baseline --steps 20 > gpurun_out/bench_C6.log 2>&1
python bench.py --config G3 --no-cpu-baseline --steps 20 > gpurun_out/bench_G3.log 2>&1
python bench.py --mode stream --steps 40 > gpurun_out/bench_C5.log 2>&1
python bench.py --mode stream --u16 --steps 40 > gpurun_out/bench_C5u16.log 2>&1
python bench.py --impl reference --steps 10 --warmup 2 > gpurun_out/bench_ref.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
