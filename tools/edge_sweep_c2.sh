for R in 1.4 1.6 1.8 2.0 2.3; do
  for C in C2 C3; do
    FLMISR_EDGE_RATIO=$R python bench.py --config $C --steps 30 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$C ratio $R', round(d['value'],1), round(d['kernels']['scg_loop']['avg_ms'],4))"
  done
done
