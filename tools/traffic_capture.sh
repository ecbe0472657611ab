# ncu --set full of the loop kernel launched by bench.py itself (bench inputs, its first launch) for every
# bench config, raw page as CSV text; dram bytes per launch -> profiles/traffic.json (tools/traffic_update.py)
for C in C2 C3 C4 C6 G3; do
  K=k_scg_loop; [ $C = G3 ] && K=k_scg_loop4
  ncu --set full --clock-control none -k regex:${K} -c 1 --csv --page raw \
      python bench.py --config $C --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/traffic_$C.csv 2>&1
done
