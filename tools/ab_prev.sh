# A/B of the current library against the previous commit's (build_variants/lib_prev.so), same box
one() { python bench.py --config $2 --no-cpu-baseline --steps 30 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2', round(d['value'],1), round(d['kernels']['scg_loop']['avg_ms'],4))" >> gpurun_out/ab_prev.txt; }
for rep in 1 2; do
  for C in C2 C3; do
    FLMISR_LIB=$PWD/build_variants/lib_prev.so one prev $C
    one new $C
  done
done
timeout 600 python -m pytest tests/test_gpu_det.py -q -x > gpurun_out/det_tests.log 2>&1; echo "exit=$?" >> gpurun_out/det_tests.log
