# 512-row band (C3 at g = 8) per-phase time vs the minimum segment length
for S in 4 7 10 13; do
  echo "SEG_MIN=$S"; FLMISR_SEG_MIN=$S python tools/band_size.py --config C3 --reps 10 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k: round(v['us_per_phase'],2) for k,v in d.items() if k.startswith('g')})"
done
