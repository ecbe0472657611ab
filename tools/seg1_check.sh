# any-length segments (partial last unrolled group): border-ratio sweep vs the previous library, then parity suites
one() { python bench.py --config $2 --no-cpu-baseline --steps $3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2', round(d['value'],1), round(d['kernels']['scg_loop']['avg_ms'],4))" >> gpurun_out/seg1_sweep.txt; }
for C in C2 C3; do
  FLMISR_LIB=$PWD/build_variants/lib_prev.so one prev $C 30
  for R in 1.3 1.4 1.5 1.6 1.7; do FLMISR_EDGE_RATIO=$R one "ratio$R" $C 30; done
  FLMISR_LIB=$PWD/build_variants/lib_prev.so one prev $C 30
done
FLMISR_LIB=$PWD/build_variants/lib_prev.so one prev C4 10
for R in 1.5 1.6 1.7 1.8; do FLMISR_EDGE_RATIO=$R one "ratio$R" C4 10; done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bands.py tests/test_gpu_e2e_oracle.py tests/test_gpu_det.py -q -x > gpurun_out/seg1_tests.log 2>&1; echo "exit=$?" >> gpurun_out/seg1_tests.log
