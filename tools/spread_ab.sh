# A/B: edge-strip items spread over the warp slots (new) vs clustered in the last CTAs (cur), same box
one() { python bench.py --config $2 --no-cpu-baseline --steps $3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2', round(d['value'],1), round(d['kernels']['scg_loop']['avg_ms'],4))" >> gpurun_out/spread_ab.txt; }
for rep in 1 2; do
  for C in C2 C3 G3; do
    FLMISR_LIB=$PWD/build_variants/lib_cur.so one cur $C 20
    one new $C 20
  done
done
FLMISR_LIB=$PWD/build_variants/lib_cur.so one cur C4 10
one new C4 10
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bands.py tests/test_gpu_e2e_oracle.py tests/test_gpu_det.py tests/test_gpu_pc.py -q -x > gpurun_out/spread_tests.log 2>&1; echo "exit=$?" >> gpurun_out/spread_tests.log
