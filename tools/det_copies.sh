timeout 900 python -m pytest tests/test_gpu_det.py tests/test_gpu_bands.py tests/test_gpu_threads.py -q -x > gpurun_out/detc_tests.log 2>&1; echo "exit=$?" >> gpurun_out/detc_tests.log
one() { python bench.py --config $2 --no-cpu-baseline --steps $3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2', round(d['value'],1), round(d['kernels']['scg_loop']['avg_ms'],4))" >> gpurun_out/detc_ab.txt; }
for C in C2 C3; do FLMISR_LIB=$PWD/build_variants/lib_cur.so one cur $C 20; one new $C 20; done
