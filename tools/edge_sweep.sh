# border-piece ratio sweep (FLMISR_EDGE_RATIO) per config: proj/s and loop ms
for R in 1.7 2.0 2.3 2.7; do
  for C in C4 G3; do
    FLMISR_EDGE_RATIO=$R python bench.py --config $C --steps 20 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$C ratio $R', round(d['value'],1), round(d['kernels']['scg_loop']['avg_ms'],4))"
  done
done
for R in 1.4 1.7 2.0; do
  FLMISR_EDGE_RATIO=$R python bench.py --config C6 --steps 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C6 ratio $R', round(d['value'],1), round(d['kernels']['scg_loop']['avg_ms'],4))"
done
