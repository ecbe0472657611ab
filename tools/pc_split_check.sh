# border-mask split of the per-phase kernels: A/B against the joint border code + G3 ratio sweep (one GPU)
python -m pytest tests/test_gpu_pc.py -q -x > gpurun_out/split_tests.log 2>&1; echo "exit=$?" >> gpurun_out/split_tests.log
one() { python bench.py --config G3 --steps 20 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(d['value'],2), round(d['kernels']['scg_loop']['avg_ms'],4))" >> gpurun_out/split_sweep.txt; }
for rep in 1 2; do
for R in 1.8 2.0 2.3 2.6 3.0; do
  FLMISR_EDGE_RATIO=$R one "split ratio $R"
  FLMISR_PC_JOINT_BORDER=1 FLMISR_EDGE_RATIO=$R one "joint ratio $R"
done
done
