timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/fxsum_tests.log 2>&1; echo "exit=$?" >> gpurun_out/fxsum_tests.log
one() { python bench.py --config $2 --no-cpu-baseline --steps $3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2', round(d['value'],1), round(d['kernels']['scg_loop']['avg_ms'],4))" >> gpurun_out/fxsum_ab.txt; }
for rep in 1 2; do
  for C in C2 G3; do
    FLMISR_LIB=$PWD/build_variants/lib_cur.so one cur $C 20
    one new $C 20
  done
done
